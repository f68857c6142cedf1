"""Regenerates tests/golden/ref_vectors.json from the UNMODIFIED reference.

Builds oracle/_ref/ref_driver from /root/reference/proj/include (read-only,
g++ on the headers as they lie; see oracle/Makefile) and captures its JSON.
Run in the build container (the GPU box has no /root/reference):

    python tests/golden/make_golden.py
"""
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))


def main() -> int:
    if not os.path.isdir("/root/reference/proj/include"):
        print("reference not present; nothing to regenerate", file=sys.stderr)
        return 1
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "_ref/ref_driver"],
                   check=True)
    out = subprocess.run([os.path.join(ROOT, "oracle", "_ref", "ref_driver"), "golden"],
                         check=True, capture_output=True, text=True).stdout
    data = json.loads(out)
    data["_generated_by"] = ("oracle/_ref/ref_driver golden (reference headers "
                             "/root/reference/proj/include, compiled read-only)")
    with open(os.path.join(HERE, "ref_vectors.json"), "w") as f:
        json.dump(data, f, separators=(",", ":"))
        f.write("\n")
    print("wrote", os.path.join(HERE, "ref_vectors.json"), len(out), "bytes")
    return 0


if __name__ == "__main__":
    sys.exit(main())
