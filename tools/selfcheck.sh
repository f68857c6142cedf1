# Self-check (stands in for compute-sanitizer, closed on this GPU pool): the same
# deterministic workload under the default and the checked library (device asserts +
# barrier jitter), with fresh memory poisoned by different patterns, with both kernel
# choices; every digest of a parameter set must be identical.
mkdir -p gpurun_out
OUT=gpurun_out/selfcheck.txt
: > $OUT
make -s -C paper_2407_19871_b200/csrc variant V=checked DEFS="-DLPB_CHECKS=1 -DLPB_JITTER=1" > /dev/null 2>&1
CHECKED=$PWD/paper_2407_19871_b200/lib_checked.so
for level in 128 80; do
  for small in 1 0; do
    for lib in default checked; do
      for poison in none 0xDEADBEEF 0x7FF80001; do
        L=""; [ $lib = checked ] && L=$CHECKED
        P=""; [ $poison != none ] && P=$poison
        line=$(LOCPIR_B200_LIB=$L LOCPIR_B200_POISON=$P LOCPIR_B200_SMALL=$small \
               timeout 600 python tools/selfcheck_run.py $level 2>&1 | tail -1)
        rc=$?
        echo "level=$level small=$small lib=$lib poison=$poison rc=$rc $line" >> $OUT
      done
    done
  done
done
python - <<'PY' >> $OUT
import collections
d = collections.defaultdict(set)
bad = 0
for ln in open("gpurun_out/selfcheck.txt"):
    if "digest" not in ln:
        bad += ln.startswith("level=")
        continue
    lv = ln.split()[0]
    d[lv].add(ln.split()[-1])
print("SUMMARY", {k: len(v) for k, v in d.items()}, "runs without a digest:", bad)
print("PASS" if bad == 0 and all(len(v) == 1 for v in d.values()) and len(d) == 2 else "FAIL")
PY
