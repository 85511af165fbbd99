"""Summarise an ncu report: per-kernel duration, DRAM bytes, throughput, occupancy."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "smsp__inst_executed.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
idx = [(w, hdr.index(w)) for w in want if w in hdr]
for r in rows[2:]:
    d = {w: r[i] for w, i in idx}
    name = d["Kernel Name"].split("(")[0].replace("void kb::<unnamed>::", "")[:28]
    t = float(d["gpu__time_duration.sum"]) * 1e-9
    rb, wb = float(d["dram__bytes_read.sum"]), float(d["dram__bytes_write.sum"])
    print(f"{name:28s} {t*1e6:9.1f}us rd {rb/1e6:8.1f}MB wr {wb/1e6:8.1f}MB  {(rb+wb)/t/1e9:7.0f}GB/s "
          f"dram% {float(d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed']):5.1f} "
          f"sm% {float(d['sm__throughput.avg.pct_of_peak_sustained_elapsed']):5.1f} "
          f"regs {d['launch__registers_per_thread']} warps% {float(d['sm__warps_active.avg.pct_of_peak_sustained_active']):5.1f} "
          f"grid {d['launch__grid_size']} inst {float(d['smsp__inst_executed.sum'])/1e6:.1f}M "
          + " ".join(f"{k.split('.')[0][-22:]}={float(d[k]):.1f}" for k in d if 'fp64' in k))
