# Round-2 (final build) capture of the latency kernels on one cfg1 query (80-bit) and on
# a 128-bit 148-gate level; each ncu pass runs only after the same command exited 0.
mkdir -p gpurun_out
timeout 300 python tools/cfg1_once.py > gpurun_out/k1l_plain.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:'lat|split|reduce' -c 6 \
  -o gpurun_out/k1l_prof python tools/cfg1_once.py > gpurun_out/k1l_ncu.log 2>&1; echo k1l=$? > gpurun_out/k1l_status.txt
python tools/ncu_summary.py gpurun_out/k1l_prof.ncu-rep > gpurun_out/k1l_summary.txt 2>&1
python tools/ncu_lines.py gpurun_out/k1l_prof.ncu-rep k_blind_rotate_lat >> gpurun_out/k1l_summary.txt 2>&1
cat gpurun_out/k1l_status.txt
