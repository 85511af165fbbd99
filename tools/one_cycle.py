"""Run exactly K restart cycles (max_iters = 60K) of one configuration —
for ncu launch lists and sanitizer runs (dev tool)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2402_15033_b200 as kb  # noqa: E402


def main():
    grid = int(sys.argv[1]) if len(sys.argv) > 1 else 512
    kind = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    cycles = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    dims = int(sys.argv[4]) if len(sys.argv) > 4 else 2
    op = kb.Laplace2D(grid, grid) if dims == 2 else kb.Laplace3D(grid, grid, grid)
    b = op.spmv(np.ones(op.n))
    shat = 60 if kind == 3 else 0
    rep = kb.sstep_gmres(op, b, None, kb.SolverConfig(scheme=kb.OrthoScheme(kb.OrthoKind(kind), shat), big_step=shat,
                                                      max_iters=60 * cycles))
    print(rep.iterations, rep.restarts, rep.cycle_residuals[:3], rep.telemetry["gpu_launches"])


if __name__ == "__main__":
    main()
