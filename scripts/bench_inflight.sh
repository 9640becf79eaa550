cd $GRAFT_REPO_ROOT
for f in ${FRAMES:-1 2 3 4}; do
  timeout 600 python bench.py --steps 60 --warmup 5 --no-e2e --no-train --no-cpu --no-c5 --inflight $f 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('== inflight $f', round(d['value'],1), 'FPS', round(d['ms_per_step'],4), 'ms/frame')
"
done
