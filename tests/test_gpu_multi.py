"""Multi-GPU parity (needs ≥ 2 visible GPUs; skipped on a 1-GPU box).

Launches tests/dist_parity.py with torchrun at N = 2 (and N = 4 when four
GPUs are visible): row-partitioned solves with NCCL halos and one Gram
allreduce per BCGS-PIP must match the reference's golden reports — through
NCCL (default) and through the one-shot NVLink peer-memory allreduce."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("peer", ["1", "0"])  # one-shot NVLink peer allreduce (k_peer.cu) / ncclAllReduce
@pytest.mark.parametrize("nranks", [2, 4])
def test_row_partitioned_solves_match_reference(kb, nranks, peer, tmp_path):
    if kb.device_count() < nranks:
        pytest.skip(f"needs {nranks} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nranks}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()),
           os.path.join(ROOT, "tests", "dist_parity.py")]
    out_dir = tmp_path / "ranks"
    out_dir.mkdir()
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env={**os.environ, "KRY_DIST_OUT": str(out_dir), "KRY_PEER_ALLREDUCE": peer})
    assert p.returncode == 0, (p.stdout[-3000:], p.stderr[-3000:])
    lines = [json.loads(f.read_text()) for f in sorted(out_dir.glob("rank*.json"))]
    assert len(lines) == nranks and all(l["ok"] for l in lines), lines
    # one Gram allreduce per BCGS-PIP plus scalar norms: the collective count is positive on every rank
    assert all(r["allreduces"] > 0 for l in lines for r in l["results"].values() if "allreduces" in r)
    assert all(r["bitwise"] for l in lines for r in l["results"].values() if "bitwise" in r)
