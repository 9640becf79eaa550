#!/bin/bash
# Sanitizers + extended fuzz + repeated exhaustive renders on the current code (evidence for profiles/).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool python scripts/sanitize.py > gpurun_out/san_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|Error SUMMARY' gpurun_out/san_$tool.log | tail -1)"
done
timeout 1500 python scripts/fuzz_many.py 2000 150 > gpurun_out/fuzz.log 2>&1; echo "fuzz rc=$?"; tail -3 gpurun_out/fuzz.log
for i in $(seq 1 20); do timeout 120 python -m pytest tests -q -m gpu -k exhaustive -x > /dev/null 2>&1 || echo "exhaustive rep $i failed"; done; echo "exhaustive reps done"
