timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "pre_keyswitch or bit_exact or mux or truth or loc_pir or comparator or city" > gpurun_out/k1l_t.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/k1l_t.log
for i in 1 2; do
timeout 600 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --gates 592 --locpir sample --locpir-configs cfg1,cfg3 > gpurun_out/k1l_b$i.log 2>&1
python - $i <<'PY'
import json,sys
d=json.loads(open(f'gpurun_out/k1l_b{sys.argv[1]}.log').read().strip().splitlines()[-1])
print(' '.join(f"{k}={x['queries_per_s']:.3f}" for k,x in d['locpir'].items() if isinstance(x,dict) and 'queries_per_s' in x), d['correct'])
PY
done
