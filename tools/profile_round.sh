# ncu captures for profiles/ (one GPU): plain runs first (must exit 0), then ncu.
set -x
B="python bench.py --gates 4736 --steps 1 --warmup 1 --no-cpu-baseline --no-locpir"
timeout 300 $B > gpurun_out/p_plain1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_blind_rotate$|^k_keyswitch$" -c 2 \
  -o gpurun_out/prof_main $B > gpurun_out/p_ncu1.log 2>&1
echo main=$? > gpurun_out/pstatus.txt
L="python tools/cfg1_once.py"
timeout 300 $L > gpurun_out/p_plain2.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"lat|split|reduce" -c 3 \
  -o gpurun_out/prof_lat $L > gpurun_out/p_ncu2.log 2>&1
echo lat=$? >> gpurun_out/pstatus.txt
timeout 300 env LOCPIR_B200_BR=warp $B > gpurun_out/p_plain3.log 2>&1 && \
  timeout 900 env LOCPIR_B200_BR=warp ncu --set full --clock-control none --import-source on -k regex:"blind_rotate_w" -c 1 \
  -o gpurun_out/prof_warp $B > gpurun_out/p_ncu3.log 2>&1
echo warp=$? >> gpurun_out/pstatus.txt
