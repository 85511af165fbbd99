"""One two-stage restart cycle at a given grid (ncu target)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2402_15033_b200 as kb
g = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
kind = int(sys.argv[2]) if len(sys.argv) > 2 else 3
op = kb.Laplace2D(g, g)
b = op.spmv(np.ones(op.n))
cfg = kb.SolverConfig(scheme=kb.OrthoScheme(kb.OrthoKind(kind), 60), max_iters=60)
rep = kb.sstep_gmres(op, b, None, cfg)
print("ok", rep.iterations, rep.cycle_residuals)
