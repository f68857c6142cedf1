"""Copy a tools/round_evidence.sh run (gpurun_out/e_*) into the committed profiles/ files:
bench lines, reference arm, ncu launch list, DRAM traffic per launch, GPU test log, and
ncu summaries (metrics + top source lines) of K1 and K2t."""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")


TAG = sys.argv[1] if len(sys.argv) > 1 else "r02"


def main():
    d = json.loads(open(os.path.join(G, "e_bench.json")).read().strip().splitlines()[-1])
    loc = {k: d.pop(k) for k in ("locpir", "cpu_baseline_locpir", "reference_standin_locpir") if k in d}
    json.dump(d, open(os.path.join(P, f"{TAG}_bench_b200.json"), "w"), indent=1)
    json.dump(loc, open(os.path.join(P, f"{TAG}_bench_b200_locpir.json"), "w"), indent=1)
    json.dump(json.loads(open(os.path.join(G, "e_ref.json")).read().strip().splitlines()[-1]),
              open(os.path.join(P, f"{TAG}_bench_reference.json"), "w"), indent=1)
    for src, dst in (("e_launches.csv", f"{TAG}_launches.csv"), ("e_gpu_tests.log", f"{TAG}_gpu_tests.log")):
        open(os.path.join(P, dst), "w").write(open(os.path.join(G, src)).read())
    rows = list(csv.reader(open(os.path.join(G, "e_traffic.csv"))))
    hdr, ks = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            x = dict(zip(hdr, r))
            key = "k_blind_rotate<3, 7>" if "blind_rotate" in x["Kernel Name"] else "k_keyswitch_tc"
            ks.setdefault(key, {})[x["Metric Name"]] = float(x["Metric Value"].replace(",", ""))
    t = {"what": "DRAM bytes read + written and L2 hit rate per launch, steady state (the first "
                 "two launches skipped), cfg2 full size (65,536 gates)",
         "command": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,"
                    "gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none "
                    "-k regex:'^k_blind_rotate$|^k_keyswitch_tc$' --launch-skip 2 -c 2 python "
                    "bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-locpir",
         "kernels": ks}
    json.dump(t, open(os.path.join(P, f"{TAG}_traffic.json"), "w"), indent=1)
    for rep, out, title in (("e_prof_br", f"{TAG}_ncu_blind_rotate.txt", "^k_blind_rotate$"),
                            ("e_prof_ks", f"{TAG}_ncu_keyswitch.txt", "^k_keyswitch_tc$")):
        r = os.path.join(G, rep + ".ncu-rep")
        summ = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_summary.py"), r],
                              capture_output=True, text=True).stdout
        src = subprocess.run(["ncu", "-i", r, "--page", "source", "--print-source", "cuda,sass", "--csv"],
                             capture_output=True, text=True, errors="replace").stdout
        open("/tmp/_src.csv", "w").write(src)
        lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), "/tmp/_src.csv"],
                               capture_output=True, text=True).stdout.splitlines()[:26]
        size = ("--gates 4736 --steps 1 --warmup 1" if rep == "e_prof_br" else
                "--steps 1 --warmup 1 (cfg2 size, --launch-skip 1)")
        hdr_line = (f"# ncu --set full --clock-control none --import-source on -k regex:'{title}' -c 1 "
                    f"python bench.py {size} --no-cpu-baseline --no-locpir\n")
        open(os.path.join(P, out), "w").write(hdr_line + summ + "\n# top CUDA source lines by warp-stall samples\n"
                                              + "\n".join(lines) + "\n")
    print("profiles updated")


if __name__ == "__main__":
    main()
