# session-5 evidence on the restored build: GPU tests, default bench (wall time recorded),
# the wall-budget fallback, the reference arm, smoke
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/m_gpu_tests.log 2>&1; echo tests=$? > gpurun_out/m_status.txt
tail -2 gpurun_out/m_gpu_tests.log >> gpurun_out/m_status.txt
S=$(date +%s)
timeout 2400 python bench.py > gpurun_out/m_bench.json 2> gpurun_out/m_bench.err; echo bench=$? wall_s=$(( $(date +%s) - S )) >> gpurun_out/m_status.txt
S=$(date +%s)
timeout 900 python bench.py --wall-budget 150 --locpir-configs cfg5 --no-cpu-baseline > gpurun_out/m_bench_budget.json 2> gpurun_out/m_bench_budget.err; echo budget=$? wall_s=$(( $(date +%s) - S )) >> gpurun_out/m_status.txt
timeout 1200 python bench.py --impl reference > gpurun_out/m_ref.json 2> gpurun_out/m_ref.err; echo ref=$? >> gpurun_out/m_status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m_smoke.log 2>&1; echo smoke=$? >> gpurun_out/m_status.txt
cat gpurun_out/m_status.txt
