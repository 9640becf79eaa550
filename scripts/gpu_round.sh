#!/bin/bash
# One GPU session: smoke, GPU tests, stage times, bench line, launch list.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 180 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q --timeout 300 -rA > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
grep -E "PASSED|FAILED|ERROR|passed|failed" gpurun_out/pytest_gpu.log | tail -40
timeout 300 python scripts/stage_times.py > gpurun_out/stage_times.log 2>&1; echo "stages rc=$?"; tail -2 gpurun_out/stage_times.log
if [ "${BENCH:-1}" = "1" ]; then
  timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.log 2>&1; echo "bench rc=$?"; tail -c 3000 gpurun_out/bench.log
fi
if [ "${LAUNCHES:-1}" = "1" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python scripts/profile_frame.py --frames 4 --backward > gpurun_out/launches.log 2>&1; echo "launch list rc=$?"
fi
