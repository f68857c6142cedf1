mkdir -p gpurun_out
timeout 2400 python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_full.log 2>&1; echo bench=$? > gpurun_out/status2.txt
