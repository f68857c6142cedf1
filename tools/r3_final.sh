# final-build check: GPU tests + the default bench line (updates profiles/r02_bench_* and
# r02_gpu_tests.log through tools/update_profiles.py --bench-only)
mkdir -p gpurun_out
make -s -C paper_2407_19871_b200/csrc > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/f_gpu_tests.log 2>&1; echo tests=$? > gpurun_out/f_status.txt
timeout 2400 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; echo bench=$? >> gpurun_out/f_status.txt
tail -2 gpurun_out/f_gpu_tests.log >> gpurun_out/f_status.txt
cat gpurun_out/f_status.txt
