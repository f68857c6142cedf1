timeout 400 python -m pytest tests/test_gpu_parity.py -q -x -k "keyswitch" > gpurun_out/kstc_tests.log 2>&1
echo "tests rc=$?" ; tail -1 gpurun_out/kstc_tests.log
for v in base kb4 base kb4; do
  if [ "$v" = base ]; then lib=""; else lib=$PWD/paper_2407_19871_b200/lib_$v.so; fi
  LOCPIR_B200_LIB=$lib timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-locpir > gpurun_out/kb_$v.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/kb_$v.log').read().strip().splitlines()[-1]);k=d['keyswitch'];print('$v','value',round(d['value']),'ks_ms',round(k['avg_launch_ms'],3),'tensor_frac',round(k['tensor_view']['frac'],3),'correct',d['correct'])"
done
