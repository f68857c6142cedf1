timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "keyswitch" > gpurun_out/kstc_tests.log 2>&1
echo "tests rc=$?" ; tail -2 gpurun_out/kstc_tests.log
for i in 1 2; do timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-locpir > gpurun_out/kb_$i.log 2>&1
python -c "
import json;d=json.loads(open('gpurun_out/kb_$i.log').read().strip().splitlines()[-1]);k=d['keyswitch'];print('value',round(d['value']),'ks_ms',round(k['avg_launch_ms'],3),'tensor_frac',round(k['tensor_view']['frac'],3),'correct',d['correct'])"; done
