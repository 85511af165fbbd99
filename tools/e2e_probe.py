"""Where the e2e step (host buffers through kry_sstep_gmres) spends its time
beyond the device-resident cycle (development aid): wall time of one
restart cycle at 4000² via the device entry point and via the host-buffer
entry point, plus the bare PCIe copies of the same bytes."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2402_15033_b200 as kb  # noqa: E402

g = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
ctx = kb.get_context()
ctx.set_timing(os.environ.get("TIMING", "1") == "1")
op = kb.Laplace2D(g, g)
n = op.n
ones = torch.ones(n, dtype=torch.float64, device="cuda")
b = torch.empty(n, dtype=torch.float64, device="cuda")
x = torch.zeros(n, dtype=torch.float64, device="cuda")
kb.lib().kry_spmv_device(ctx.handle, op.handle, ones.data_ptr(), b.data_ptr())
cfg = kb.SolverConfig(scheme=kb.OrthoScheme(kb.OrthoKind(3), 60), big_step=60, max_iters=60)
hb = torch.empty(n, dtype=torch.float64, pin_memory=True)
hx = torch.zeros(n, dtype=torch.float64, pin_memory=True)
torch.cuda.synchronize()
hb.copy_(b.cpu())
P = lambda t: C.cast(C.c_void_p(t.data_ptr()), kb._capi.P_dbl)  # noqa: E731
ccfg = cfg.to_c()


def dev():
    kb.sstep_gmres_device(op, b.data_ptr(), x.data_ptr(), cfg, x.data_ptr())


def host():
    rep_c, cyc, pb, pbp = kb._new_report(1024)
    kb._check(kb.lib().kry_sstep_gmres(ctx.handle, op.handle, P(hb), P(hx), C.byref(ccfg), C.byref(rep_c), P(hx)))


def copies():
    b.copy_(hb, non_blocking=True)
    x.copy_(hx, non_blocking=True)
    hx.copy_(x, non_blocking=True)
    torch.cuda.synchronize()


for name, fn in (("device cycle", dev), ("host cycle", host), ("pcie copies", copies), ("device cycle", dev)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    print(f"{name:14s} {1e3 * (time.perf_counter() - t) / 10:8.3f} ms")
