# full round check on one B200: GPU tests, smoke, bench (with CPU baseline), reference arm,
# ncu launch list of the bench command
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? > gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/status.txt
tail -5 gpurun_out/gpu_tests.log >> gpurun_out/status.txt
timeout 600 python bench.py > gpurun_out/bench_full.log 2>&1; echo bench=$? >> gpurun_out/status.txt
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo ref=$? >> gpurun_out/status.txt
timeout 300 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain_launch.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo launches=$? >> gpurun_out/status.txt
