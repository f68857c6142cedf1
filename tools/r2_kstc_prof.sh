# K2t profile: full ncu capture at 4,736 gates + DRAM traffic at cfg2 size (steady state)
S="python bench.py --gates 4736 --steps 1 --warmup 1 --no-cpu-baseline --no-locpir"
timeout 300 $S > gpurun_out/kp_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^k_keyswitch_tc$" -c 1 \
  -o gpurun_out/kp_ks $S > gpurun_out/kp_ncu.log 2>&1; echo ks=$?
B1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-locpir"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,lts__t_bytes.sum \
  --clock-control none -k regex:"^k_keyswitch_tc$" --launch-skip 1 -c 2 --csv --log-file gpurun_out/kp_traffic.csv $B1 > gpurun_out/kp_traffic.log 2>&1; echo traffic=$?
