#!/bin/bash
# Repeat one test with a long per-test timeout; sample GPU utilisation while it runs.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in $(seq 1 ${REPS:-8}); do
  t0=$(date +%s)
  timeout -k 10 ${LIMIT:-200} python -m pytest ${FILES} -q -x --timeout ${PT:-180} --timeout-method thread -p no:cacheprovider --durations=3 > gpurun_out/s2_$i.log 2>&1 &
  pid=$!
  while kill -0 $pid 2>/dev/null; do sleep 10; el=$(( $(date +%s)-t0 )); if [ $el -gt 40 ]; then echo "rep $i t=$el util=$(nvidia-smi --query-gpu=utilization.gpu,clocks.sm,power.draw --format=csv,noheader)"; fi; done
  wait $pid; rc=$?; echo "rep $i rc=$rc $(( $(date +%s)-t0 ))s $(grep -E 'passed|failed' gpurun_out/s2_$i.log | tail -1)"; grep -A3 "slowest" gpurun_out/s2_$i.log | tail -3
done
