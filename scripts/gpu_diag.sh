#!/bin/bash
# Diagnosis run: the failing GPU tests, then the bench legs one at a time with wall-clock times.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 400 python -m pytest tests/test_gpu_exhaustive.py tests/test_gpu_device_api.py -q -x --timeout 200 > gpurun_out/diag_pt.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/diag_pt.log
for leg in "--no-e2e --no-train --no-c5 --no-cpu --no-c1" "--no-e2e --no-train --no-cpu --no-c1" "--no-train --no-c5 --no-cpu --no-c1" "--no-e2e --no-c5 --no-cpu --no-c1"; do
  t0=$(date +%s); timeout 300 python bench.py --steps 10 --warmup 3 $leg > gpurun_out/diag_b.log 2>&1; rc=$?; t1=$(date +%s)
  echo "bench [$leg] rc=$rc $((t1-t0))s"; grep '^{' gpurun_out/diag_b.log | python -c "import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k:d.get(k) for k in ('value','latency_ms_per_frame','fwd_bwd_ms_per_view')}, (d.get('c5') or {}).get('ms_per_frame'), (d.get('e2e') or {}).get('value'), (d.get('train_step') or {}).get('ms_per_step'), d.get('frame',{}).get('fixup_pixels'))"
done
