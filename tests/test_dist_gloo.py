"""Multi-rank host logic on the CPU (world_size 2 and 8, gloo, 127.0.0.1).

The B200 path partitions rows across ranks (kry_laplace_partition: whole
grid lines / planes), exchanges one halo line/plane with each neighbour
before every SpMV, and allreduces the (c0+w)×w Gram once per BCGS-PIP; the
small factorizations are then replicated on every rank.  These tests run that
protocol with gloo in place of NCCL: the product's own partition function,
the same halo send/recv pattern, a numpy restatement of the stencil kernel's
neighbour selection (local row vs halo plane), and the product's host
Cholesky (kry_try_cholesky) on the allreduced Gram — which must yield
bit-identical factors on every rank (identical control decisions)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def partition(kb, dims, nx, ny, nz, nranks, rank):
    rb, nl, h = C.c_int64(), C.c_int64(), C.c_int64()
    rc = kb.lib().kry_laplace_partition(dims, nx, ny, nz, nranks, rank, C.byref(rb), C.byref(nl), C.byref(h))
    assert rc == 0, kb.lib().kry_last_error()
    return rb.value, nl.value, h.value


def local_stencil(dims, nx, ny, nz, rb, nl, x, lo, hi):
    """numpy restatement of stencil_kernel's neighbour selection (k_ops.cu)."""
    y = np.empty(nl)
    plane = nx * ny
    for i in range(nl):
        row = rb + i

        def at(col):
            if col < rb:
                return lo[col - (rb - (nx if dims == 2 else plane))]
            if col >= rb + nl:
                return hi[col - (rb + nl)]
            return x[col - rb]

        s = 0.0
        if dims == 2:
            iy, ix = divmod(row, nx)
            terms = [(iy > 0, -1.0, row - nx), (ix > 0, -1.0, row - 1), (True, 4.0, row),
                     (ix + 1 < nx, -1.0, row + 1), (iy + 1 < ny, -1.0, row + nx)]
        else:
            iz, rem = divmod(row, plane)
            iy, ix = divmod(rem, nx)
            terms = [(iz > 0, -1.0, row - plane), (iy > 0, -1.0, row - nx), (ix > 0, -1.0, row - 1),
                     (True, 6.0, row), (ix + 1 < nx, -1.0, row + 1), (iy + 1 < ny, -1.0, row + nx),
                     (iz + 1 < nz, -1.0, row + plane)]
        for ok, c, col in terms:
            if ok:
                s = s + c * at(col)
        y[i] = s
    return y


def worker(rank, world, port, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import sys
        sys.path.insert(0, ROOT)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import paper_2402_15033_b200 as kb
        from oracle import orc
        out = {}
        for dims, (nx, ny, nz) in [(2, (13, max(11, 2 * world + 1), 1)), (3, (7, 6, max(5, world + 1)))]:
            rb, nl, h = partition(kb, dims, nx, ny, nz, world, rank)
            n = nx * ny * (nz if dims == 3 else 1)
            a = orc.laplace2d(nx, ny) if dims == 2 else orc.laplace3d(nx, ny, nz)
            x = np.random.default_rng(7).standard_normal(n)
            xl = x[rb:rb + nl].copy()
            lo, hi = np.zeros(h), np.zeros(h)
            # the product's halo pattern (kb_operator.cpp): first h rows to rank-1, last h rows to rank+1
            reqs = []
            if rank > 0:
                reqs.append(dist.isend(torch.from_numpy(xl[:h].copy()), rank - 1))
                t = torch.zeros(h, dtype=torch.float64)
                dist.recv(t, rank - 1)
                lo = t.numpy()
            if rank + 1 < world:
                reqs.append(dist.isend(torch.from_numpy(xl[nl - h:].copy()), rank + 1))
                t = torch.zeros(h, dtype=torch.float64)
                dist.recv(t, rank + 1)
                hi = t.numpy()
            for r in reqs:
                r.wait()
            y = local_stencil(dims, nx, ny, nz, rb, nl, xl, lo, hi)
            out[f"spmv{dims}"] = bool(np.array_equal(y, orc.spmv(a, x)[rb:rb + nl]))
            out[f"range{dims}"] = (rb, nl)
        # distributed Gram + replicated Cholesky
        rng = np.random.default_rng(11)
        n = 1000
        Q, _ = np.linalg.qr(rng.standard_normal((n, 10)))
        V = rng.standard_normal((n, 6))
        rb, nl = rank * n // world, (rank + 1) * n // world - rank * n // world
        Xl = np.hstack([Q, V])[rb:rb + nl]
        G = torch.from_numpy(Xl.T @ V[rb:rb + nl])
        dist.all_reduce(G)
        G = G.numpy()
        gl = np.hstack([Q, V]).T @ V
        out["gram_err"] = float(np.abs(G - gl).max() / np.abs(gl).max())  # relative
        rcol, gvv = G[:10], G[10:]
        S = gvv - rcol.T @ rcol
        R, piv = kb.try_cholesky(S)
        allR = [torch.zeros(36, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allR, torch.from_numpy(np.ascontiguousarray(R).reshape(-1)))
        out["chol_identical"] = all(torch.equal(allR[0], t) for t in allR)
        out["pivot"] = piv
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as e:  # surface the failure to the parent
        q.put((rank, {"error": repr(e)}))


@pytest.mark.parametrize("world", [2, 8])  # 8: the driver's largest one-node run (bench.py --gpus 8)
def test_multi_rank_partition_halo_gram_protocol(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r in range(world):
        assert "error" not in res[r], res[r]
        assert res[r]["spmv2"] and res[r]["spmv3"]
        assert res[r]["gram_err"] < 1e-12
        assert res[r]["chol_identical"] and res[r]["pivot"] == 0
    # the partition tiles the rows exactly, in rank order
    for d, n in [(2, 13 * max(11, 2 * world + 1)), (3, 7 * 6 * max(5, world + 1))]:
        nxt = 0
        for r in range(world):
            b, nl = res[r][f"range{d}"]
            assert b == nxt and nl > 0
            nxt = b + nl
        assert nxt == n


def test_partition_errors():
    import paper_2402_15033_b200 as kb
    rb, nl, h = C.c_int64(), C.c_int64(), C.c_int64()
    assert kb.lib().kry_laplace_partition(2, 10, 3, 1, 4, 0, C.byref(rb), C.byref(nl), C.byref(h)) != 0
    assert kb.lib().kry_laplace_partition(2, 10, 8, 1, 3, 2, C.byref(rb), C.byref(nl), C.byref(h)) == 0
    assert (rb.value, nl.value, h.value) == (50, 30, 10)
