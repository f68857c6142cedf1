# K2s split A/B on latency-bound levels (cfg1 circuits): adaptive split (default build) vs
# the fixed 32-way split (lib_ks32.so)
mkdir -p gpurun_out
L=paper_2407_19871_b200
for v in default ks32 default ks32; do
  if [ $v = default ]; then lib=$PWD/$L/liblocpir_b200.so; else lib=$PWD/$L/lib_$v.so; fi
  LOCPIR_B200_LIB=$lib timeout 300 python tools/latency_check.py 2>&1 | sed "s/^/$v /" >> gpurun_out/ks_ab.log
done
timeout 900 python -m pytest tests -m gpu -x -q -k "keyswitch or latency or cfg1 or city or exact or small or maj" >> gpurun_out/ks_ab.log 2>&1; echo tests=$? >> gpurun_out/ks_ab.log
cat gpurun_out/ks_ab.log
