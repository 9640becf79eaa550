# e2e (host f64 API) throughput vs the host-staging knobs: "threads raw_fraction scalar" triples
python -m pytest tests/test_gpu_device_api.py -x -q -m gpu -k narrowing 2>&1 | tail -1
for cfg in ${E2E_CFGS:-16,0.1,0 8,0.1,0 12,0.1,0 16,0.2,0 12,0.05,0 16,0.1,0}; do
  set -- $(echo $cfg | tr , " ")
  if [ "$3" = 1 ]; then export GEER_HOST_SCALAR=1; else unset GEER_HOST_SCALAR; fi
  GEER_HOST_THREADS=$1 GEER_HOST_RAW_FRACTION=$2 timeout 600 python bench.py --steps 10 --warmup 3 --no-train --no-c5 --no-c1 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('threads $1 raw $2 scalar $3:', round(d['value']), round(e['value'],1), round(e['ms_per_step'],2), round(e['fwd_bwd']['ms_per_view'],2))"
done
