# compute-sanitizer, ONE tool per gpurun call: bash tools/sanitize.sh memcheck|racecheck|synccheck
# Runs tools/sanitize_run.py twice (small-level kernels, then LOCPIR_B200_SMALL=0 for the
# throughput kernels K1/K2) after a plain run of the same command exited 0.
TOOL=${1:-memcheck}
mkdir -p gpurun_out
OUT=gpurun_out/san_$TOOL.txt
echo "== compute-sanitizer --tool $TOOL" > $OUT
for SMALL in 1 0; do
  timeout 300 env LOCPIR_B200_SMALL=$SMALL python tools/sanitize_run.py >> $OUT 2>&1 || { echo "plain run failed" >> $OUT; exit 1; }
  timeout 1800 env LOCPIR_B200_SMALL=$SMALL compute-sanitizer --tool $TOOL --print-limit 20 \
      python tools/sanitize_run.py >> $OUT 2>&1
  echo "SMALL=$SMALL rc=$?" >> $OUT
done
