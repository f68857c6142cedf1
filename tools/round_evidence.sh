# Round-end evidence on one GPU: GPU tests, the default bench line, the reference arm,
# the ncu launch list of the bench command, DRAM traffic per launch, full captures of
# K1/K2.  Every ncu pass runs only after the same command exited 0 without ncu.
set -x
make -s -C paper_2407_19871_b200/csrc > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/e_gpu_tests.log 2>&1; echo tests=$? > gpurun_out/e_status.txt
timeout 2400 python bench.py > gpurun_out/e_bench.json 2> gpurun_out/e_bench.err; echo bench=$? >> gpurun_out/e_status.txt
timeout 1200 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/e_ref.json 2> gpurun_out/e_ref.err; echo ref=$? >> gpurun_out/e_status.txt
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-locpir"
timeout 600 $B > gpurun_out/e_plain.json 2>&1 && \
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/e_launches.csv $B > gpurun_out/e_ncu_launch.log 2>&1; echo launches=$? >> gpurun_out/e_status.txt
B1="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-locpir"
# steady state: skip the warm-up launches (the first one streams the BK into L2 cold)
timeout 1500 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
  --clock-control none -k regex:"^k_blind_rotate$|^k_keyswitch_tc$" --launch-skip 2 -c 2 --csv --log-file gpurun_out/e_traffic.csv $B1 > gpurun_out/e_ncu_traffic.log 2>&1; echo traffic=$? >> gpurun_out/e_status.txt
S="python bench.py --gates 4736 --steps 1 --warmup 1 --no-cpu-baseline --no-locpir"
timeout 300 $S > gpurun_out/e_plain_small.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_blind_rotate$" -c 1 \
  -o gpurun_out/e_prof_br $S > gpurun_out/e_ncu_br.log 2>&1; echo br=$? >> gpurun_out/e_status.txt
# K2t at cfg2 size (at 4,736 gates its grid is only 1.3 waves)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"^k_keyswitch_tc$" --launch-skip 1 -c 1 \
  -o gpurun_out/e_prof_ks $B1 > gpurun_out/e_ncu_ks.log 2>&1; echo ks=$? >> gpurun_out/e_status.txt
cat gpurun_out/e_status.txt
