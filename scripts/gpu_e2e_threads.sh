# e2e (host f64 API) throughput vs the host-staging knobs: threads x raw fraction
python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -x -q -m gpu 2>&1 | tail -2
for cfg in "16 0" "16 0.15" "16 0.25" "16 0.35" "16 0.5" "8 0.35" "16 1.0"; do
  set -- $cfg
  GEER_HOST_THREADS=$1 GEER_HOST_RAW_FRACTION=$2 timeout 600 python bench.py --steps 10 --warmup 3 --no-train --no-c5 --no-c1 --no-cpu 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', round(d['value']), round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],2))"
done
