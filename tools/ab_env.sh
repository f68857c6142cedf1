# A/B over an environment variable: bash tools/ab_env.sh VAR value1 value2 ...
var=$1; shift
echo "" > gpurun_out/ab.txt
for v in "$@"; do
  env $var=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "bit_exact or mux" > gpurun_out/ab_${v}_tests.log 2>&1
  echo "$var=$v tests rc=$? $(tail -1 gpurun_out/ab_${v}_tests.log)" >> gpurun_out/ab.txt
  env $var=$v timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-locpir > gpurun_out/ab_$v.log 2>&1
  python - "$v" <<'PY' >> gpurun_out/ab.txt
import json, sys
v = sys.argv[1]
try:
    d = json.loads(open(f'gpurun_out/ab_{v}.log').read().strip().splitlines()[-1])
    print('%-10s value %.0f ms/step %.1f br_ms %.1f frac %.3f ks_ms %.1f e2e %.0f correct %s' % (v, d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['keyswitch']['avg_launch_ms'], d['e2e']['value'], d['correct']))
except Exception as e:
    print(v, 'FAILED', e, open(f'gpurun_out/ab_{v}.log').read()[-500:])
PY
done
