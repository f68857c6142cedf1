# (1) K2t input-load cache hint A/B: time + DRAM traffic at cfg2 for base and kef
for v in base kef; do
  if [ "$v" = base ]; then lib=""; else lib=$PWD/paper_2407_19871_b200/lib_$v.so; fi
  LOCPIR_B200_LIB=$lib timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    --clock-control none -k regex:"^k_keyswitch_tc$" --launch-skip 1 -c 2 --csv --log-file gpurun_out/kt_$v.csv \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-locpir > gpurun_out/kt_$v.log 2>&1; echo $v=$?
  LOCPIR_B200_LIB=$lib timeout 300 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-locpir > gpurun_out/ktb_$v.log 2>&1
done
# (2) K1l on one cfg1 query: launch list + one full capture
timeout 300 python tools/cfg1_once.py > gpurun_out/k1l_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k1l_launches.csv python tools/cfg1_once.py > gpurun_out/k1l_l.log 2>&1; echo launches=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_blind_rotate_lat" --launch-skip 3 -c 1 \
  -o gpurun_out/k1l_prof python tools/cfg1_once.py > gpurun_out/k1l_ncu.log 2>&1; echo k1l=$?
