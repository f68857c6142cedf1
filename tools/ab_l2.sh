bash tools/ab_bench.sh noel
cp gpurun_out/ab.txt gpurun_out/ab1.txt
bash tools/ab_env.sh LOCPIR_B200_L2PERSIST 0
cat gpurun_out/ab1.txt gpurun_out/ab.txt > gpurun_out/ab_all.txt
