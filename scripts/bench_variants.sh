cd $GRAFT_REPO_ROOT
for defs in "$@"; do
  GEER_NVCC_DEFS="$defs" python -m paper_2505_24053_b200.build --force > /dev/null 2>&1 || { echo "build failed: $defs"; continue; }
  timeout 600 python bench.py --steps 50 --warmup 5 --no-e2e --no-train --no-cpu --no-c5 $BENCH_ARGS 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('== $defs', round(d['value'],1), 'FPS', round(d['fwd_bwd_ms_per_view'],3), 'fb_ms', {k:round(v['ms'],3) for k,v in d['stages'].items()})
"
done
