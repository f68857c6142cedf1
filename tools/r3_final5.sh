# final evidence on the last build: self-check, GPU tests, default bench line, reference arm
mkdir -p gpurun_out
make -s -C paper_2407_19871_b200/csrc > /dev/null; make -s -C oracle all > /dev/null
bash tools/selfcheck.sh > /dev/null 2>&1; tail -2 gpurun_out/selfcheck.txt > gpurun_out/k_status.txt
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/k_gpu_tests.log 2>&1; echo tests=$? >> gpurun_out/k_status.txt
timeout 2400 python bench.py > gpurun_out/k_bench.json 2> gpurun_out/k_bench.err; echo bench=$? >> gpurun_out/k_status.txt
timeout 1200 python bench.py --impl reference > gpurun_out/k_ref.json 2> gpurun_out/k_ref.err; echo ref=$? >> gpurun_out/k_status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/k_smoke.log 2>&1; echo smoke=$? >> gpurun_out/k_status.txt
tail -2 gpurun_out/k_gpu_tests.log >> gpurun_out/k_status.txt
cat gpurun_out/k_status.txt
