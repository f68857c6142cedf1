# final evidence on the last build: GPU tests, the default bench line, the shard emulation
mkdir -p gpurun_out
make -s -C paper_2407_19871_b200/csrc > /dev/null
timeout 1800 python -m pytest tests -m gpu -q -s > gpurun_out/g_gpu_tests.log 2>&1; echo tests=$? > gpurun_out/g_status.txt
timeout 2400 python bench.py > gpurun_out/g_bench.json 2> gpurun_out/g_bench.err; echo bench=$? >> gpurun_out/g_status.txt
timeout 2400 python bench.py --steps 3 --warmup 1 --no-cpu-baseline --locpir sample --emulate-shards > gpurun_out/g_emul.json 2> gpurun_out/g_emul.err; echo emul=$? >> gpurun_out/g_status.txt
tail -2 gpurun_out/g_gpu_tests.log >> gpurun_out/g_status.txt
cat gpurun_out/g_status.txt
