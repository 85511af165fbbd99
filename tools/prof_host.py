"""Host-side latency profile of full solves (KRY_HOST_PROFILE=1 prints the
time blocked in stream syncs per solve): 512² to convergence and one 4000²
cycle, two-stage ŝ = 60."""
import os, sys, time
os.environ.setdefault("KRY_HOST_PROFILE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2402_15033_b200 as kb

ctx = kb.get_context()
for g, iters in [(512, 500000), (4000, 60)]:
    op = kb.Laplace2D(g, g, ctx)
    one = torch.ones(op.n, dtype=torch.float64, device="cuda")
    b = torch.empty_like(one)
    x = torch.zeros_like(one)
    torch.cuda.synchronize()
    kb.lib().kry_spmv_device(ctx.handle, op.handle, one.data_ptr(), b.data_ptr())
    cfg = kb.SolverConfig(scheme=kb.OrthoScheme(kb.OrthoKind.TWO_STAGE, 60), big_step=60, max_iters=iters)
    for rep_i in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        rep = kb.sstep_gmres_device(op, b.data_ptr(), None, cfg, x.data_ptr())
        torch.cuda.synchronize()
        print(f"grid {g} run {rep_i}: {time.perf_counter() - t0:.4f} s, {rep.restarts + 1} cycles, "
              f"{rep.iterations} its, status {rep.status.name}", flush=True)
    del op
