# ncu --set full of K1 (k_blind_rotate<3,7>) and K2 (k_keyswitch) on a 4,736-gate batch (32 CTAs/SM)
mkdir -p gpurun_out
B="python bench.py --gates 4736 --steps 1 --warmup 1 --no-cpu-baseline --no-locpir"
timeout 300 $B > gpurun_out/p_plain1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_blind_rotate$|^k_keyswitch$" -s 2 -c 2 \
  -o gpurun_out/prof_r2a $B > gpurun_out/p_ncu1.log 2>&1
echo main=$? > gpurun_out/pstatus.txt
