timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status.txt
python - <<'PY' >> gpurun_out/status.txt
import json
d=json.loads(open('gpurun_out/bench.log').read().strip().splitlines()[-1])
print('value %.0f ms/step %.1f br_ms %.1f frac %.3f ks_ms %.1f e2e %.0f correct %s' % (d['value'], d['ms_per_step'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['keyswitch']['avg_launch_ms'], d['e2e']['value'], d['correct']))
PY
