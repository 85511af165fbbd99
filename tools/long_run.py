"""Sustained-run probe: per-cycle device time over a long loop of 8000² cycles,
with nvidia-smi sampled alongside (SM / memory clocks, power, throttle
reasons).  Prints one JSON line (dev tool)."""
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2402_15033_b200 as kb  # noqa: E402


def main():
    grid = int(sys.argv[1]) if len(sys.argv) > 1 else 8000
    cycles = int(sys.argv[2]) if len(sys.argv) > 2 else 100
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=timestamp,clocks.sm,clocks.mem,power.draw,"
                            "clocks_event_reasons.active,temperature.gpu", "--format=csv,noheader,nounits",
                            "-lms", "500"], stdout=subprocess.PIPE, text=True)
    ctx = kb.get_context()
    op = kb.Laplace2D(grid, grid, ctx)
    one = torch.ones(op.n, dtype=torch.float64, device="cuda")
    b = torch.empty_like(one)
    x = torch.zeros_like(one)
    torch.cuda.synchronize()
    kb.lib().kry_spmv_device(ctx.handle, op.handle, one.data_ptr(), b.data_ptr())
    cfg = kb.SolverConfig(scheme=kb.OrthoScheme(kb.OrthoKind.TWO_STAGE, 60), big_step=60, max_iters=60)
    ts = []
    for _ in range(cycles):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        kb.sstep_gmres_device(op, b.data_ptr(), x.data_ptr(), cfg, x.data_ptr())
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    smi.terminate()
    out, _ = smi.communicate()
    print(json.dumps({"grid": grid, "cycles": cycles, "ms_per_cycle_by_decile":
                      [round(sum(ts[i:i + cycles // 10]) / (cycles // 10), 2) for i in range(0, cycles, cycles // 10)],
                      "smi": out.splitlines()[::4]}))


if __name__ == "__main__":
    main()
