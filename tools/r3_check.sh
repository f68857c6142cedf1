mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? > gpurun_out/status.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/status.txt
tail -3 gpurun_out/gpu_tests.log >> gpurun_out/status.txt
timeout 400 python bench.py --steps 5 --warmup 3 --locpir sample > gpurun_out/bench.log 2>&1; echo bench=$? >> gpurun_out/status.txt
tail -c 3000 gpurun_out/bench.log >> gpurun_out/status.txt
