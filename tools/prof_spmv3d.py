"""Repeated 3-D stencil SpMVs at a given grid (ncu target)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2402_15033_b200 as kb
g = int(sys.argv[1]) if len(sys.argv) > 1 else 256
op = kb.Laplace3D(g, g, g)
x = np.ones(op.n)
for _ in range(3):
    y = op.spmv(x)
print("ok", float(y[:10].sum()))
