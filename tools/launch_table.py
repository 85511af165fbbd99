"""Per-family table of the last restart cycle in an ncu launch list, and the
bench's `roofline.traffic` figures (profiles/ncu_traffic.json).

usage: python tools/launch_table.py LAUNCHES.csv [--traffic-out profiles/ncu_traffic.json --key-suffix @4000x4000]

The launch list is `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum --clock-control none --csv` over `bench.py --steps 1
--warmup 1` (two cycles: warm-up + timed); the last cycle is the launches
after the last-but-one `xupdate_kernel` (the cycle-closing solution update)."""
import argparse
import collections
import csv
import json
import re


def load(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    h = rows[0]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    launches = collections.OrderedDict()
    for r in rows[1:]:
        d = launches.setdefault(r[ii], {"name": re.sub(r"\(.*", "", r[ki]).replace("void ", "")
                                        .replace("kb::<unnamed>::", "")})
        d[r[mi]] = float(r[vi].replace(",", ""))
    return list(launches.values())


def family(name):
    if name.startswith("gram_kernel"):
        return "gram_kernel"
    if name.startswith("update_"):  # update_kernel, update_tma_kernel, update_mma_kernel
        return "update_kernel"
    return name


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csv")
    ap.add_argument("--traffic-out")
    ap.add_argument("--key-suffix", default="@4000x4000")
    a = ap.parse_args()
    L = load(a.csv)
    ends = [i for i, d in enumerate(L) if d["name"].startswith("xupdate_kernel")]
    start = ends[-2] + 1 if len(ends) >= 2 else 0
    cyc = L[start:ends[-1] + 1] if ends else L
    fam = collections.OrderedDict()
    for d in cyc:
        f = fam.setdefault(d["name"], [0, 0.0, 0.0, 0.0])
        f[0] += 1
        f[1] += d["gpu__time_duration.sum"] * 1e-6
        f[2] += d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
    tot = sum(f[1] for f in fam.values())
    print(f"| kernel | launches | time (ms) | share | DRAM bytes (GB) | DRAM GB/s |")
    print("|---|---|---|---|---|---|")
    for n, (c, t, b, _) in sorted(fam.items(), key=lambda kv: -kv[1][1]):
        print(f"| {n} | {c} | {t:.3f} | {100 * t / tot:.1f} % | {b / 1e9:.2f} | {b / 1e9 / (t * 1e-3):.0f} |")
    print(f"| **total** | {sum(f[0] for f in fam.values())} | {tot:.3f} | | | |")
    if a.traffic_out:
        per = collections.defaultdict(list)
        for d in cyc:
            per[family(d["name"])].append(d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"])
        out = {f"{k}{a.key_suffix}": sum(v) / len(v) for k, v in per.items() if k in ("gram_kernel", "update_kernel")}
        out["_source"] = (f"{a.csv} (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
                          "--clock-control none over `bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e "
                          "--no-tts512`); mean DRAM bytes per launch of the family over the timed restart cycle")
        try:
            old = json.load(open(a.traffic_out))
        except (OSError, ValueError):
            old = {}
        src = old.pop("_source", None)
        old.update(out)
        if src and src != out["_source"]:
            old["_source"] = f"{out['_source']}; earlier keys: {src}"
        with open(a.traffic_out, "w") as f:
            json.dump(old, f, indent=1)
        print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
