import sys, time
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2402_15033_b200 as kb
for grid in (512, 2000):
    ctx = kb.get_context()
    op = kb.Laplace2D(grid, grid, ctx)
    one = torch.ones(op.n, dtype=torch.float64, device="cuda"); b = torch.empty_like(one); x = torch.zeros_like(one)
    kb.lib().kry_spmv_device(ctx.handle, op.handle, one.data_ptr(), b.data_ptr())
    for label, knd, sh in [("standard", None, 0), ("two_stage", kb.OrthoKind.TWO_STAGE, 60), ("pip2", kb.OrthoKind.BCGS_PIP2, 0)]:
        cfg = kb.SolverConfig(scheme=kb.OrthoScheme(knd or kb.OrthoKind.BCGS_PIP2, sh), big_step=sh, max_iters=600)
        fn = kb.standard_gmres_device if knd is None else kb.sstep_gmres_device
        fn(op, b.data_ptr(), None, cfg, x.data_ptr())
        torch.cuda.synchronize(); t = time.perf_counter()
        rep = fn(op, b.data_ptr(), None, cfg, x.data_ptr())
        torch.cuda.synchronize(); dt = time.perf_counter() - t
        print(grid, label, f"{dt*1e3/ (rep.restarts + 1):.3f} ms/cycle", rep.iterations, rep.restarts, flush=True)
