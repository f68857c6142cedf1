# final bench line + reference arm on the last build
mkdir -p gpurun_out
make -s -C paper_2407_19871_b200/csrc > /dev/null; make -s -C oracle all > /dev/null
timeout 2400 python bench.py > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err; echo bench=$? > gpurun_out/i_status.txt
timeout 1200 python bench.py --impl reference > gpurun_out/i_ref.json 2> gpurun_out/i_ref.err; echo ref=$? >> gpurun_out/i_status.txt
cat gpurun_out/i_status.txt
