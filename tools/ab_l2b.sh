echo "" > gpurun_out/ab.txt
for cfg in "noel 0" "noel 1" "base 0" "base 1"; do
  set -- $cfg; v=$1; lp=$2
  if [ "$v" = base ]; then lib=""; else lib=$PWD/paper_2407_19871_b200/lib_$v.so; fi
  LOCPIR_B200_LIB=$lib LOCPIR_B200_L2PERSIST=$lp timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-locpir > gpurun_out/ab_x.log 2>&1
  python - "$v L2PERSIST=$lp" <<'PY' >> gpurun_out/ab.txt
import json, sys
d = json.loads(open('gpurun_out/ab_x.log').read().strip().splitlines()[-1])
print('%-22s value %.0f br_ms %.1f frac %.3f ks_ms %.1f' % (sys.argv[1], d['value'], d['roofline']['avg_launch_ms'], d['roofline']['frac'], d['keyswitch']['avg_launch_ms']))
PY
done
