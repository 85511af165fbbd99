"""One line per bench.py JSON file: value, ms/step, e2e, roofline frac,
scheme / ŝ (development aid for profiles/README.md)."""
import json
import sys

for f in sys.argv[1:]:
    try:
        lines = [ln for ln in open(f).read().splitlines() if ln.startswith("{")]
        d = json.loads(lines[-1])
    except (OSError, IndexError, ValueError) as e:
        print(f"{f}: {e}")
        continue
    c = d.get("config", {})
    e2e = d.get("e2e") or {}
    rf = d.get("roofline") or {}
    print(f"{f.split('/')[-1]:40s} N={d.get('n_gpus')} value={d.get('value', 0):8.0f} ms/step={d.get('ms_per_step', 0):7.2f} "
          f"e2e={e2e.get('value', 0):6.0f} frac={rf.get('frac', 0):.3f} kernel={rf.get('kernel', '')} "
          f"{c.get('workload', '')[:60]}")
