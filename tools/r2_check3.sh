mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? > gpurun_out/status3.txt
timeout 1800 python -m pytest tests -m gpu -x -q -s > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/status3.txt
tail -3 gpurun_out/gpu_tests.log >> gpurun_out/status3.txt
grep "FFT rounding margin" gpurun_out/gpu_tests.log >> gpurun_out/status3.txt
timeout 600 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --locpir sample > gpurun_out/bench_q.log 2>&1; echo bench=$? >> gpurun_out/status3.txt
