"""Merge reference outputs produced elsewhere (tools/golden_box.sh on the GPU
box host) into tests/golden/solver_golden.json, exactly as make_golden.py's
merge() does (TEST INFRASTRUCTURE).
usage: python tools/golden_merge.py REF.json FMA.json
       python tools/golden_merge.py REF.json --no-fma   (the FMA build's run did not fit in
       memory: the envelope is taken as zero, i.e. the strict 1e-10 relative
       per-cycle tolerance, and the entry is marked "fma_unavailable")"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from make_golden import merge  # noqa: E402


def main():
    ref = json.load(open(sys.argv[1]))
    no_fma = sys.argv[2] == "--no-fma"
    res = {"ref": ref, "fma": ref if no_fma else json.load(open(sys.argv[2]))}
    path = os.path.join(ROOT, "tests", "golden", "solver_golden.json")
    golden = json.load(open(path))
    merge(golden, res)
    if no_fma:
        for k in ref:
            golden[k]["fma_unavailable"] = True
    with open(path, "w") as f:
        json.dump(golden, f, indent=1)
    for k in res["ref"]:
        g = golden[k]
        print("merged", k, g["status"], g["iterations"], g["restarts"], g["reduces"], g["cycle_residuals"])


if __name__ == "__main__":
    main()
