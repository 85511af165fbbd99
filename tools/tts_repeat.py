import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2402_15033_b200 as kb
ctx = kb.get_context()
g = int(sys.argv[1]) if len(sys.argv) > 1 else 512
op = kb.Laplace2D(g, g, ctx)
one = torch.ones(op.n, dtype=torch.float64, device="cuda"); b = torch.empty_like(one); x = torch.zeros_like(one)
torch.cuda.synchronize()
kb.lib().kry_spmv_device(ctx.handle, op.handle, one.data_ptr(), b.data_ptr())
cfg = kb.SolverConfig(scheme=kb.OrthoScheme(kb.OrthoKind.TWO_STAGE, 60), big_step=60)
ts = []
for i in range(6):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    rep = kb.sstep_gmres_device(op, b.data_ptr(), None, cfg, x.data_ptr())
    torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
print(os.environ.get("KRY_FUSED_MPK"), g, ["%.4f" % t for t in ts], rep.iterations)
