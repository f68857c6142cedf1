timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "cfg2_full or gates_bit_exact or truth" > gpurun_out/pipe_tests.log 2>&1
echo "tests rc=$?"; tail -1 gpurun_out/pipe_tests.log
for v in 4 0 8 4; do
  LOCPIR_B200_PIPE_CHUNKS=$v timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-locpir > gpurun_out/pipe_$v.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/pipe_$v.log').read().strip().splitlines()[-1]);print('chunks $v','value',round(d['value']),'e2e',round(d['e2e']['value']),'ks',round(d['keyswitch']['avg_launch_ms'],3),'correct',d['correct'])"
done
