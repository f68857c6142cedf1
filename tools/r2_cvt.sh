timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/cvt_tests.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/cvt_tests.log
for i in 1 2; do timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-locpir > gpurun_out/cvt_b$i.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/cvt_b$i.log').read().strip().splitlines()[-1]);print('value',round(d['value']),'br_ms',round(d['roofline']['avg_launch_ms'],1),'frac',round(d['roofline']['frac'],3),'e2e',round(d['e2e']['value']),'correct',d['correct'])"; done
timeout 600 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --gates 592 --locpir sample --locpir-configs cfg1 > gpurun_out/cvt_c1.log 2>&1
python - <<'PY'
import json
d=json.loads(open('gpurun_out/cvt_c1.log').read().strip().splitlines()[-1])
for k,x in d['locpir'].items():
    if isinstance(x,dict) and 'queries_per_s' in x: print(k, round(x['queries_per_s'],3), x.get('correct'))
PY
