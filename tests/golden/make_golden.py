"""Generate the golden fixtures under tests/golden/ from the CPU reference.

TEST INFRASTRUCTURE.  Runs the unmodified reference (oracle/_ref, compiled in
place from /root/reference by oracle/Makefile) in this container and writes:

  solver_golden.json   per solver config: the reference SolveReport
                       (status, iterations, restarts, reduces, SyncCounter
                       deltas, per-cycle residuals, final residual) for the
                       reference's own Release build AND for the same
                       reference compiled with FMA contraction.  |ref − fma|
                       per cycle is the reference's own rounding envelope;
                       the GPU parity tolerance is 10× that.
  kernels_golden.npz   small fixed inputs/outputs: SpMV (5-pt, 7-pt, CSR),
                       MPK, gram, BCGS-PIP, BCGS-PIP2, try_cholesky, a
                       store sequence (R, Q) and a Hessenberg/LSQ solve.

Usage: make -C oracle ref ref_fma && python tests/golden/make_golden.py
"""
import json
import os
import subprocess
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

# (key, grid, dims, kind, shat, standard, operator, x0 value, max_iters)
SOLVER_CONFIGS = [
    ("pip2_2d16", 16, 2, 2, 0, False, "stencil", None, 500000),
    ("pip2_2d64", 64, 2, 2, 0, False, "stencil", None, 500000),
    ("pip2_2d100", 100, 2, 2, 0, False, "stencil", None, 500000),
    ("two_2d64_s60", 64, 2, 3, 60, False, "stencil", None, 500000),
    ("two_2d100_s60", 100, 2, 3, 60, False, "stencil", None, 500000),
    ("two_2d100_s20", 100, 2, 3, 20, False, "stencil", None, 500000),
    ("two_2d100_s30", 100, 2, 3, 30, False, "stencil", None, 500000),
    ("two_2d100_s5", 100, 2, 3, 5, False, "stencil", None, 500000),
    ("two_2d128_s60", 128, 2, 3, 60, False, "stencil", None, 500000),
    ("two_3d16_s60", 16, 3, 3, 60, False, "stencil", None, 500000),
    ("standard_2d32", 32, 2, 1, 0, True, "stencil", None, 500000),
    ("two_2d48_csr", 48, 2, 3, 60, False, "csr", None, 500000),
    ("pip2_2d64_warm", 64, 2, 2, 0, False, "stencil", 0.5, 120),
    ("two_2d200_s60", 200, 2, 3, 60, False, "stencil", None, 500000),
    ("pip2_2d128", 128, 2, 2, 0, False, "stencil", None, 500000),
    # BASELINE-size configs (round 2).  configs[0] full solves at 512²; a
    # multi-cycle 3-D golden (64³ needs 3 restarts); configs[1]/[2] as
    # exactly-k-cycle runs through max_iters = 60k (SURVEY §8(c) "Large configs").
    ("pip2_2d512", 512, 2, 2, 0, False, "stencil", None, 500000),
    ("two_2d512_s60", 512, 2, 3, 60, False, "stencil", None, 500000),
    ("two_3d64_s60", 64, 3, 3, 60, False, "stencil", None, 500000),
    ("pip2_3d64", 64, 3, 2, 0, False, "stencil", None, 500000),
    ("two_3d64_s20", 64, 3, 3, 20, False, "stencil", None, 500000),
    ("two_2d4000_s60_c2", 4000, 2, 3, 60, False, "stencil", None, 120),
    ("pip2_2d4000_c2", 4000, 2, 2, 0, False, "stencil", None, 120),
    ("two_2d8000_s60_c1", 8000, 2, 3, 60, False, "stencil", None, 60),
    # BASELINE configs[4] at n = 20,000 (grid = n): the random-sparse
    # generator (oracle/randsparse.py ≡ kry_gen_random_sparse, diag_factor
    # 0.15, 30 entries per row), Jacobi-scaled: the reference is handed D⁻¹A
    # and D⁻¹b with b = A·1 (5-6 restarts).
    ("rand20k_two_s60_jac", 20000, 0, 3, 60, False, "random", None, 500000),
    ("rand20k_pip2_jac", 20000, 0, 2, 0, False, "random", None, 500000),
    ("rand20k_two_s20_jac", 20000, 0, 3, 20, False, "random", None, 500000),
]
# Configs whose CPU reference run takes minutes (generated with --only, merged).
LARGE = {"pip2_2d512", "two_2d512_s60", "two_2d4000_s60_c2", "pip2_2d4000_c2", "two_2d8000_s60_c1"}


def solve_all(only=None):
    import time
    from oracle import ref
    out = {}
    for key, g, dims, kind, shat, standard, opk, x0v, mi in SOLVER_CONFIGS:
        if only is not None and key not in only:
            continue
        t0 = time.perf_counter()
        if opk == "random":
            a, b = random_jacobi_system(g)
        else:
            a = ref.laplace2d(g, g) if dims == 2 else ref.laplace3d(g, g, g)
            b = ref.spmv(a, np.ones(a.n))
        x0 = None if x0v is None else np.full(a.n, x0v)
        rep = ref.solve(a, b, x0, ref.make_config(kind=kind, big_step=shat, shat=shat, max_iters=mi),
                        standard=standard)
        out[key] = {
            "grid": g, "dims": dims, "kind": kind, "shat": shat, "standard": standard, "operator": opk,
            "x0": x0v, "max_iters": mi,
            "status": rep.status, "iterations": rep.iterations, "restarts": rep.restarts,
            "reduces": rep.reduces, "per_block": [int(v) for v in rep.per_block],
            "per_big_panel": [int(v) for v in rep.per_big_panel],
            "cycle_residuals": [float(v) for v in rep.cycle_residuals],
            "initial_residual": rep.initial_residual,
            "final_relative_residual": rep.final_relative_residual,
            "breakdown": rep.breakdown,
            "reference_seconds": time.perf_counter() - t0,
        }
    return out


def random_jacobi_system(n, per_row=30, seed=1, diag_factor=0.15):
    """(D⁻¹A, D⁻¹b), b = A·1, of the configs[4] generator — what the device
    path computes with kry_operator_jacobi on A and the original b."""
    from oracle import ref, randsparse
    rp, ci, vv = randsparse.random_sparse(n, 0, n, per_row, seed, diag_factor)
    a = ref.Csr(n, rp, ci, vv)
    b = ref.spmv(a, np.ones(n))
    d = vv[np.nonzero(ci == np.repeat(np.arange(n), np.diff(rp)))[0]]
    rps, cis, vvs = randsparse.random_sparse(n, 0, n, per_row, seed, diag_factor, jacobi=True)
    return ref.Csr(n, rps, cis, vvs), b / d


def kernels():
    from oracle import ref
    rng = np.random.default_rng(20240226)
    d = {}
    a2 = ref.laplace2d(9, 7)
    x2 = rng.standard_normal(a2.n)
    d["lap2d_9x7_x"], d["lap2d_9x7_y"] = x2, ref.spmv(a2, x2)
    a3 = ref.laplace3d(5, 4, 3)
    x3 = rng.standard_normal(a3.n)
    d["lap3d_5x4x3_x"], d["lap3d_5x4x3_y"] = x3, ref.spmv(a3, x3)
    d["lap2d_9x7_rowptr"], d["lap2d_9x7_col"], d["lap2d_9x7_val"] = a2.row_ptr, a2.col_idx, a2.vals
    start = rng.standard_normal(a2.n)
    d["mpk_start"], d["mpk_V"] = start, ref.mpk(a2, start, 5)
    q, _ = np.linalg.qr(rng.standard_normal((257, 11)))
    q = np.asfortranarray(q)
    v = rng.standard_normal((257, 6))
    d["pip_q"], d["pip_v"] = q, v
    qq, rc, rj, red = ref.bcgs_pip(q, v)
    d["pip_out_q"], d["pip_out_rcol"], d["pip_out_rjj"] = qq, rc, rj
    qq2, rc2, rj2, _ = ref.bcgs_pip2(q, v)
    d["pip2_out_q"], d["pip2_out_rcol"], d["pip2_out_rjj"] = qq2, rc2, rj2
    d["gram_v"], d["gram_out"] = v, ref.gram(v)
    s = v.T @ v
    d["chol_s"] = s
    d["chol_r"], piv = ref.try_cholesky(s)
    d["chol_pivot"] = np.array([piv])
    s_bad = s.copy()
    s_bad[3, 3] = -1.0
    d["chol_bad_s"] = s_bad
    d["chol_bad_r"], pivb = ref.try_cholesky(s_bad)
    d["chol_bad_pivot"] = np.array([pivb])
    # a two-stage store sequence on the 12×12 Laplacian (RawSequenceReconstruction shape)
    a = ref.laplace2d(12, 12)
    b = ref.spmv(a, np.ones(a.n))
    v1 = b / np.linalg.norm(b)
    st = ref.Store(a.n, 12, 3, 12)
    blocks = []
    for j in range(4):
        blk = ref.mpk(a, v1 if j == 0 else st.column(st.info().filled - 1), 3)
        blocks.append(blk)
        st.preprocess_block(blk, j != 0)
    st.finalize_big_panel()
    d["store_blocks"] = np.stack(blocks)
    d["store_R"], d["store_Q"] = st.coefficients(), st.all()
    k = st.info().filled - 1
    d["store_H"] = st.hessenberg(k)
    y, imp, valid = ref_lsq(d["store_H"], 2.5)
    d["lsq_y"], d["lsq_implicit"] = y, np.array([imp, valid])
    return d


def ref_lsq(h, gamma):
    import ctypes as C
    from oracle import ref
    h = np.asfortranarray(h)
    k = h.shape[1]
    y = np.zeros(k)
    imp, valid = C.c_double(), C.c_int64()
    ref._chk(ref.lib().kref_hessenberg_lsq(k, ref._p(h), gamma, ref._p(y), C.byref(imp), C.byref(valid)))
    return y[: valid.value], imp.value, valid.value


def main():
    """python make_golden.py                 all small configs + kernels_golden.npz
       python make_golden.py --only k1,k2    just these solver configs, merged into solver_golden.json
       python make_golden.py --large         the LARGE set (minutes to an hour of CPU), merged"""
    if len(sys.argv) > 1 and sys.argv[1] == "--solve-json":
        only = set(sys.argv[2].split(",")) if len(sys.argv) > 2 else None
        print(json.dumps(solve_all(only)))
        return
    only = None
    if len(sys.argv) > 2 and sys.argv[1] == "--only":
        only = sys.argv[2].split(",")
    elif len(sys.argv) > 1 and sys.argv[1] == "--large":
        only = [k for k, *_ in SOLVER_CONFIGS if k in LARGE]
    elif len(sys.argv) == 1:
        only = [k for k, *_ in SOLVER_CONFIGS if k not in LARGE]
    subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), "ref", "ref_fma"], check=True)
    path = os.path.join(HERE, "solver_golden.json")
    golden = json.load(open(path)) if os.path.exists(path) else {}
    for key in only:
        # One process per key and variant; the two variants run side by side
        # unless the store (8·61·n bytes) of two of them would not fit in memory.
        grid = next(c[1] for c in SOLVER_CONFIGS if c[0] == key)
        procs = {}
        for variant in ("ref", "fma"):
            env = dict(os.environ, KRY_REF_VARIANT=variant)
            procs[variant] = subprocess.Popen([sys.executable, __file__, "--solve-json", key], env=env,
                                              stdout=subprocess.PIPE, text=True)
            if grid >= 8000:
                procs[variant].wait()
        res = {}
        for variant, pr in procs.items():
            out, _ = pr.communicate()
            if pr.returncode != 0:
                raise SystemExit(f"{key}/{variant}: reference run failed ({pr.returncode})")
            res[variant] = json.loads(out)
        merge(golden, res)
        with open(path, "w") as f:
            json.dump(golden, f, indent=1)
        print("wrote", key, golden[key]["status"], golden[key]["iterations"], golden[key]["restarts"],
              f"{golden[key]['reference_seconds']:.1f} s", flush=True)
    if len(sys.argv) == 1:
        np.savez_compressed(os.path.join(HERE, "kernels_golden.npz"), **kernels())
        print("wrote", os.path.join(HERE, "kernels_golden.npz"))


def merge(golden, res):
    for key, rep in res["ref"].items():
        fma = res["fma"][key]
        rep["fma_same_counts"] = all(rep[k] == fma[k] for k in ("iterations", "restarts", "reduces"))
        rep["fma_cycle_residuals"] = fma["cycle_residuals"]
        golden[key] = rep


if __name__ == "__main__":
    main()
