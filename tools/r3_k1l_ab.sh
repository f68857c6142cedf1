# K1l A/B: BK load placement (LAT_BK_SPREAD / LAT_BK_B0 / LAT_BK_B1) -- launch ms per level
# size (tools/br_sweep.py) and cfg1 latency (tools/latency_check.py) per library build
mkdir -p gpurun_out
L=paper_2407_19871_b200
for v in default lat0 latA latB default; do
  if [ $v = default ]; then lib=$PWD/$L/liblocpir_b200.so; else lib=$PWD/$L/lib_$v.so; fi
  LOCPIR_B200_LIB=$lib timeout 300 python tools/br_sweep.py $v 4,64,148 >> gpurun_out/k1l_ab.log 2>&1
  LOCPIR_B200_LIB=$lib timeout 300 python tools/latency_check.py 2>&1 | sed "s/^/$v /" >> gpurun_out/k1l_ab.log
done
LOCPIR_B200_LIB=$PWD/$L/lib_phclk.so timeout 300 python tools/k1l_phase.py >> gpurun_out/k1l_ab.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -k "lat or small or cfg1 or latency or city or loc_pir or exact" >> gpurun_out/k1l_ab.log 2>&1; echo tests=$? >> gpurun_out/k1l_ab.log
cat gpurun_out/k1l_ab.log
