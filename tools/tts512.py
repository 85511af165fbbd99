"""Time to solution at BASELINE configs[0] (2D Laplace 512², tol 1e-6):
median of R full solves per scheme, inputs resident in HBM (dev A/B tool)."""
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2402_15033_b200 as kb  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    grid = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    ctx = kb.get_context()
    op = kb.Laplace2D(grid, grid, ctx)
    one = torch.ones(op.n, dtype=torch.float64, device="cuda")
    b = torch.empty_like(one)
    x = torch.zeros_like(one)
    torch.cuda.synchronize()
    kb.lib().kry_spmv_device(ctx.handle, op.handle, one.data_ptr(), b.data_ptr())
    out = {}
    for label, knd, sh in [("bcgs_pip2", kb.OrthoKind.BCGS_PIP2, 0), ("two_stage_shat60", kb.OrthoKind.TWO_STAGE, 60)]:
        cfg = kb.SolverConfig(scheme=kb.OrthoScheme(knd, sh), big_step=sh)
        kb.sstep_gmres_device(op, b.data_ptr(), None, cfg, x.data_ptr())
        ts = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rep = kb.sstep_gmres_device(op, b.data_ptr(), None, cfg, x.data_ptr())
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        out[label] = (statistics.median(ts), min(ts), rep.iterations, rep.restarts, rep.final_relative_residual)
    print({k: tuple(round(v, 5) if isinstance(v, float) and v > 1e-3 else v for v in t) for k, t in out.items()},
          {k: v for k, v in os.environ.items() if k.startswith("KRY_")})


if __name__ == "__main__":
    main()
