#!/bin/bash
# Kernel times of one C2 fwd+bwd frame pair (ncu launch list) + stage times: the quick tuning loop.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
if [ -n "$GEER_NVCC_DEFS" ]; then python -m paper_2505_24053_b200.build --force > /dev/null 2>&1 || echo "build failed"; fi
timeout 200 python scripts/stage_times.py > gpurun_out/st.log 2>&1; tail -1 gpurun_out/st.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kt.csv python scripts/profile_frame.py --frames 2 --backward > /dev/null 2>&1
python scripts/summarize_launches.py gpurun_out/kt.csv | sed -n 5,12p
