# full-size (cfg2, 65,536 gates) single-launch captures for roofline.traffic (DRAM bytes/launch)
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-locpir"
timeout 600 $B > gpurun_out/t_plain.log 2>&1 && \
  timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:"^k_blind_rotate$|^k_keyswitch$" -c 2 --csv --log-file gpurun_out/traffic.csv $B > gpurun_out/t_ncu.log 2>&1
echo traffic=$? > gpurun_out/tstatus.txt
K="python bench.py --gates 4736 --steps 1 --warmup 1 --no-cpu-baseline --no-locpir"
timeout 300 $K > gpurun_out/t_plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_keyswitch$" -c 1 -o gpurun_out/prof_ks2 $K > gpurun_out/t_ncu2.log 2>&1
echo ks=$? >> gpurun_out/tstatus.txt
