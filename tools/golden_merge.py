"""Merge reference outputs produced elsewhere (tools/golden_box.sh on the GPU
box host) into tests/golden/solver_golden.json, exactly as make_golden.py's
merge() does (TEST INFRASTRUCTURE).
usage: python tools/golden_merge.py REF.json FMA.json"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
from make_golden import merge  # noqa: E402


def main():
    res = {"ref": json.load(open(sys.argv[1])), "fma": json.load(open(sys.argv[2]))}
    path = os.path.join(ROOT, "tests", "golden", "solver_golden.json")
    golden = json.load(open(path))
    merge(golden, res)
    with open(path, "w") as f:
        json.dump(golden, f, indent=1)
    for k in res["ref"]:
        g = golden[k]
        print("merged", k, g["status"], g["iterations"], g["restarts"], g["reduces"], g["cycle_residuals"])


if __name__ == "__main__":
    main()
