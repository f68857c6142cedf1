# ncu refresh on the final build (after the zero-copy gate_batch_host commit): launch list of
# the bench command, steady-state DRAM traffic, full captures of K1 / K2t.  Each ncu pass
# runs only after the same command exited 0 without ncu.  Output names match
# tools/round_evidence.sh so tools/update_profiles.py can read them.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-locpir"
timeout 600 $B > gpurun_out/e_plain.json 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/e_launches.csv $B > gpurun_out/e_ncu_launch.log 2>&1; echo launches=$? > gpurun_out/n_status.txt
B1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-locpir"
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:"^k_blind_rotate$|^k_keyswitch_tc$" --launch-skip 2 -c 2 --csv --log-file gpurun_out/e_traffic.csv $B1 > gpurun_out/e_ncu_traffic.log 2>&1; echo traffic=$? >> gpurun_out/n_status.txt
S="python bench.py --gates 4736 --steps 1 --warmup 1 --no-cpu-baseline --no-locpir"
timeout 300 $S > gpurun_out/e_plain_small.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_blind_rotate$" -c 1 \
  -o gpurun_out/e_prof_br $S > gpurun_out/e_ncu_br.log 2>&1; echo br=$? >> gpurun_out/n_status.txt
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^k_keyswitch_tc$" --launch-skip 1 -c 1 \
  -o gpurun_out/e_prof_ks $B1 > gpurun_out/e_ncu_ks.log 2>&1; echo ks=$? >> gpurun_out/n_status.txt
cat gpurun_out/n_status.txt
