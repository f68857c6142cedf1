# K1x bring-up: parity (K1x vs K1l vs oracle), latency-level tests, then cfg1 A/B
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cluster_latency or pre_keyswitch or bit_exact or mux or truth or loc_pir" > gpurun_out/k1x_tests.log 2>&1
echo "tests rc=$?"; tail -3 gpurun_out/k1x_tests.log
for v in 1 0; do
  LOCPIR_B200_CLUSTER=$v timeout 600 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --gates 592 \
     --locpir sample --locpir-configs cfg1 > gpurun_out/k1x_b$v.log 2>&1; echo "bench $v rc=$?"
  python - $v <<'PY'
import json,sys
v=sys.argv[1]
try:
    d=json.loads(open(f'gpurun_out/k1x_b{v}.log').read().strip().splitlines()[-1])
    for k,x in d['locpir'].items():
        if isinstance(x,dict) and 'queries_per_s' in x: print(v, k, round(x['queries_per_s'],2), x.get('correct'), x.get('latency_floor'))
except Exception as e:
    print(v,'FAILED',e, open(f'gpurun_out/k1x_b{v}.log').read()[-1500:])
PY
done
