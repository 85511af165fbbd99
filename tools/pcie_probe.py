"""PCIe pinned-copy bandwidth on this box (explains bench.py's e2e − value gap):
times the bench's per-step host traffic (b and x0 in: 2 × 8n bytes, x out:
8n bytes at n = 16 M) with CUDA events, best of 5."""
import torch

n = 16_000_000
h_in = torch.empty(2 * n, dtype=torch.float64, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float64, pin_memory=True)
d = torch.empty(2 * n, dtype=torch.float64, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, fn, nbytes in (("h2d", lambda: d.copy_(h_in, non_blocking=True), 16 * n),
                         ("d2h", lambda: h_out.copy_(d[:n], non_blocking=True), 8 * n)):
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{name}: {nbytes / 1e6:.0f} MB in {best:.3f} ms = {nbytes / best / 1e6:.1f} GB/s")
