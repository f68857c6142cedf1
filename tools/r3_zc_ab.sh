# zero-copy gate_batch_host A/B: previous library (copy path, lib_prev.so) vs the new one
mkdir -p gpurun_out
L=paper_2407_19871_b200
for v in prev default prev default; do
  if [ $v = default ]; then lib=$PWD/$L/liblocpir_b200.so; else lib=$PWD/$L/lib_$v.so; fi
  LOCPIR_B200_LIB=$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-locpir > gpurun_out/zc_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/zc_$v.json').read().strip().splitlines()[-1]); print('$v value %.0f e2e %.0f br_ms %.1f' % (d['value'], d['e2e']['value'], d['roofline']['avg_launch_ms']))" >> gpurun_out/zc_ab.log
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "zero_copy or full_size or truth or bit_exact" >> gpurun_out/zc_ab.log 2>&1; echo tests=$? >> gpurun_out/zc_ab.log
cat gpurun_out/zc_ab.log
