# quick GPU check: smoke, bit-exact parity subset, short bench (used with gpurun)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke=$? > gpurun_out/status.txt
timeout 600 python -m pytest tests -m gpu -x -q -k "bit_exact or mux or truth" > gpurun_out/gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/status.txt
tail -3 gpurun_out/gpu_tests.log >> gpurun_out/status.txt
bash tools/quick_bench.sh
