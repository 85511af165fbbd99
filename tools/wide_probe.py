"""Development probe: relative Q error of wide BCGS-PIP blocks vs the reference."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2402_15033_b200 as kb
from oracle import ref

rng = np.random.default_rng(3)
kb.get_context()
def orth(n, k):
    q, _ = np.linalg.qr(rng.standard_normal((n, k)))
    return np.asfortranarray(q)
for c0, w in [(0, 65), (0, 128), (0, 129), (40, 65), (40, 128), (40, 129), (64, 2), (60, 70), (0, 72)]:
    n = 2000
    q = orth(n, c0) if c0 else None
    v = rng.standard_normal((n, w))
    res = kb.bcgs_pip(q, v, kb.SyncCounter())
    q_ref, rc_ref, rj_ref, red = ref.bcgs_pip(q, v)
    e = np.linalg.norm(res.q - q_ref) / np.linalg.norm(q_ref)
    ecol = np.linalg.norm(res.q - q_ref, axis=0) / np.linalg.norm(q_ref, axis=0)
    bad = np.nonzero(ecol > 1e-10)[0]
    print(f"c0={c0:3d} w={w:3d} rel={e:.2e} bad cols {bad[:10].tolist()}{'...' if bad.size > 10 else ''} n_bad={bad.size}")
