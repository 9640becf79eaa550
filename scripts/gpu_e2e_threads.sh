# e2e (host f64 API) throughput vs the host-staging knobs: threads x raw fraction (x scalar narrowing)
python -m pytest tests/test_gpu_device_api.py -x -q -m gpu -k narrowing 2>&1 | tail -2
for cfg in ${E2E_CFGS:-"16 0.2 0" "16 0.2 1" "16 0.1 0" "16 0.3 0" "16 0 0"}; do
  set -- $cfg
  if [ "$3" = 1 ]; then export GEER_HOST_SCALAR=1; else unset GEER_HOST_SCALAR; fi
  GEER_HOST_THREADS=$1 GEER_HOST_RAW_FRACTION=$2 timeout 600 python bench.py --steps 10 --warmup 3 --no-train --no-c5 --no-c1 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('threads $1 raw $2 scalar $3:', round(d['value']), round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],2))"
done
