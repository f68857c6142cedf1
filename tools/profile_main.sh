B="python bench.py --gates 4736 --steps 1 --warmup 1 --no-cpu-baseline --no-locpir"
timeout 300 $B > gpurun_out/p_plain1.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_blind_rotate$|^k_keyswitch$" -c 2 -o gpurun_out/prof_main $B > gpurun_out/p_ncu1.log 2>&1; echo main=$? > gpurun_out/pstatus.txt
