for v in base km64 km128 km256 km512; do
  if [ "$v" = base ]; then lib=""; else lib=$PWD/paper_2407_19871_b200/lib_$v.so; fi
  LOCPIR_B200_LIB=$lib timeout 300 python tools/ks_sweep.py $v 2>&1 | tail -2
done
LOCPIR_B200_LIB=$PWD/paper_2407_19871_b200/lib_km128.so timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "keyswitch or mux or loc_pir" 2>&1 | tail -1
