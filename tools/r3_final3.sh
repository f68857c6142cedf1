# final evidence (CPU baseline lane-batched): GPU tests, default bench line, reference arm
mkdir -p gpurun_out
make -s -C paper_2407_19871_b200/csrc > /dev/null; make -s -C oracle all > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/h_gpu_tests.log 2>&1; echo tests=$? > gpurun_out/h_status.txt
timeout 2400 python bench.py > gpurun_out/h_bench.json 2> gpurun_out/h_bench.err; echo bench=$? >> gpurun_out/h_status.txt
timeout 1200 python bench.py --impl reference > gpurun_out/h_ref.json 2> gpurun_out/h_ref.err; echo ref=$? >> gpurun_out/h_status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/h_smoke.log 2>&1; echo smoke=$? >> gpurun_out/h_status.txt
tail -2 gpurun_out/h_gpu_tests.log >> gpurun_out/h_status.txt
cat gpurun_out/h_status.txt
