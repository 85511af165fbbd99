"""The CPU reference's own time to solution at 512² (BASELINE configs[0]),
measured on this machine's host cores: the unmodified reference compiled
in place (oracle/_ref/libkrylov_ref.so, test infrastructure — timed here as
the baseline, never shipped), 2-D Laplace 512², b = A·1, x0 = 0, m = 60,
s = 5, rel_tol 1e-6.

usage: KRYLOV_NUM_THREADS=T python tools/cpu_ref_tts.py {two-stage|bcgs-pip2} [grid]
Prints one JSON line (seconds = the reference's SolveReport.wall_seconds
scope, timed around the call)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import ref  # noqa: E402

scheme = sys.argv[1]
grid = int(sys.argv[2]) if len(sys.argv) > 2 else 512
a = ref.laplace2d(grid, grid)
b = ref.spmv(a, np.ones(a.n))
cfg = ref.make_config(kind=3, shat=60, big_step=60) if scheme == "two-stage" else ref.make_config(kind=2)
t = time.perf_counter()
rep = ref.solve(a, b, None, cfg)
dt = time.perf_counter() - t
print(json.dumps({"impl": "reference (oracle/_ref, unmodified headers, -O3 -DNDEBUG)", "grid": [grid, grid],
                  "scheme": scheme, "threads": int(os.environ.get("KRYLOV_NUM_THREADS", "1")),
                  "host_cores": os.cpu_count(), "seconds": dt, "status": int(rep.status),
                  "iterations": rep.iterations, "restarts": rep.restarts, "reduces": rep.reduces,
                  "final_relative_residual": rep.final_relative_residual}))
