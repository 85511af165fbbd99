"""Fused first-stage pass (K6) check at one grid size: one two-stage restart
cycle, report + telemetry (development aid; run once with KRY_FUSED_PASS=0
for the unfused reference numbers)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import paper_2402_15033_b200 as kb  # noqa: E402

g = int(sys.argv[1])
cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 1
ctx = kb.get_context()
ctx.set_timing(True)
op = kb.Laplace2D(g, g)
b = op.spmv(np.ones(op.n))
cfg = kb.SolverConfig(scheme=kb.OrthoScheme(kb.OrthoKind(3), 60), big_step=60, max_iters=60 * cycles)
t = time.time()
rep = kb.sstep_gmres(op, b, None, cfg)
T = rep.telemetry
print(f"grid {g} fused={os.environ.get('KRY_FUSED_PASS', '1')} wall {time.time() - t:.3f}s it {rep.iterations} "
      f"reduces {rep.sync.reduces} cyc {['%.10e' % c for c in rep.cycle_residuals]}")
print("  ms: ortho %.3f gram %.3f update %.3f fused %.3f mpk %.3f | fused launches %d, fused GB/s %.0f" % (
    1e3 * T['ortho_seconds'], 1e3 * T['gram_kernel_seconds'], 1e3 * T['update_kernel_seconds'],
    1e3 * T['fused_kernel_seconds'], 1e3 * T['mpk_seconds'], T['fused_launches'],
    T['fused_bytes'] / max(T['fused_kernel_seconds'], 1e-12) / 1e9))
