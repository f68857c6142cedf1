timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/fc_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/fc_tests.log
timeout 900 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --gates 592 --locpir sample --locpir-configs cfg1,cfg3 > gpurun_out/fc_b.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open('gpurun_out/fc_b.log').read().strip().splitlines()[-1])
for k,x in d['locpir'].items():
    if isinstance(x,dict) and 'queries_per_s' in x: print(k, round(x['queries_per_s'],3), x.get('correct'))
PY
bash tools/selfcheck.sh > /dev/null 2>&1; tail -2 gpurun_out/selfcheck.txt
