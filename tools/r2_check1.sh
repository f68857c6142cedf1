# round 2: smoke, world-2 sharded LocPIR on one GPU, full-size bench (no CPU baseline)
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? > gpurun_out/status.txt
timeout 900 python -m pytest tests/test_multirank_gpu.py -m gpu -x -q > gpurun_out/mr_tests.log 2>&1; echo mr=$? >> gpurun_out/status.txt
tail -3 gpurun_out/mr_tests.log >> gpurun_out/status.txt
timeout 1500 python bench.py --steps 3 --warmup 1 --no-cpu-baseline > gpurun_out/bench_full.log 2>&1; echo bench=$? >> gpurun_out/status.txt
