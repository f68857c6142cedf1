mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? > gpurun_out/status4.txt
timeout 2400 python -m pytest tests -m gpu -q -s > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/status4.txt
tail -3 gpurun_out/gpu_tests.log >> gpurun_out/status4.txt
grep -E "FFT rounding margin|FAILED|Error" gpurun_out/gpu_tests.log | head -20 >> gpurun_out/status4.txt
timeout 300 python tools/sanitize_run.py > gpurun_out/san_plain.log 2>&1; echo sanplain=$? >> gpurun_out/status4.txt
timeout 600 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --locpir sample > gpurun_out/bench_q.log 2>&1; echo bench=$? >> gpurun_out/status4.txt
