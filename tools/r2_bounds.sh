# upper bounds (results wrong by construction): K1 time without the intra-warp exchange /
# without the BK loads, against the product build
for v in base nointra nobk; do
  if [ "$v" = base ]; then lib=""; else lib=$PWD/paper_2407_19871_b200/lib_$v.so; fi
  LOCPIR_B200_LIB=$lib timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-locpir > gpurun_out/bd_$v.log 2>&1
  python -c "
import json;d=json.loads(open('gpurun_out/bd_$v.log').read().strip().splitlines()[-1]);print('$v','br_ms',round(d['roofline']['avg_launch_ms'],1),'frac',round(d['roofline']['frac'],3),'correct',d['correct'])" 2>&1 | tail -1
done
