"""Quick performance probe (development aid, not the bench)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2402_15033_b200 as kb

ctx = kb.get_context()
ctx.set_timing(True)
grids = [int(g) for g in sys.argv[1:]] or [512, 2000, 4000]
for g in grids:
    for kind, shat in [(3, 60), (2, 0)]:
        op = kb.Laplace2D(g, g)
        b = op.spmv(np.ones(op.n))
        cfg = kb.SolverConfig(scheme=kb.OrthoScheme(kb.OrthoKind(kind), shat), big_step=shat, max_iters=120)
        t = time.time()
        rep = kb.sstep_gmres(op, b, None, cfg)
        dt = time.time() - t
        T = rep.telemetry
        cyc = max(1, len(rep.cycle_residuals))
        print(f"grid {g} kind {kind} shat {shat}: wall {dt:.3f}s cycles {cyc} it {rep.iterations} "
              f"relres {rep.final_relative_residual:.3e}")
        print("   per cycle ms: mpk %.3f ortho %.3f gram %.3f update %.3f restart %.3f | wall %.3f" % tuple(
            1e3 * v / cyc for v in (T['mpk_seconds'], T['ortho_seconds'], T['gram_kernel_seconds'],
                                    T['update_kernel_seconds'], T['restart_seconds'], rep.wall_seconds)))
        print("   GB/s: ortho %.0f gram %.0f update %.0f mpk %.0f ; launches %d" % (
            T['ortho_bytes'] / max(T['ortho_seconds'], 1e-12) / 1e9,
            T['gram_bytes'] / max(T['gram_kernel_seconds'], 1e-12) / 1e9,
            T['update_bytes'] / max(T['update_kernel_seconds'], 1e-12) / 1e9,
            T['mpk_bytes'] / max(T['mpk_seconds'], 1e-12) / 1e9, T['gpu_launches']))
        del op
