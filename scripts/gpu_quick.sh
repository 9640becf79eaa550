#!/bin/bash
# Quick check: parity-critical GPU tests, stage times, kernel launch list of one forward frame.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_assoc_check.py tests/test_gpu_exhaustive.py tests/test_gpu_device_api.py -q -x --timeout 300 > gpurun_out/quick_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/quick_pytest.log
timeout 300 python scripts/stage_times.py > gpurun_out/stage_times.log 2>&1; echo "stages rc=$?"; tail -1 gpurun_out/stage_times.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q.csv python scripts/profile_frame.py --frames 2 > /dev/null 2>&1; echo "ncu rc=$?"
