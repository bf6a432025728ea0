"""Compact table of bench JSON lines."""
import json
import sys

for path in sys.argv[1:]:
    for line in open(path):
        line = line.strip()
        if not line.startswith("{"):
            continue
        d = json.loads(line)
        c = d.get("config", {})
        r = d.get("roofline") or {}
        print(f"{c.get('workload','?')[:28]:28s} {c.get('schedule','-'):9s} "
              f"value={d['value']:8.1f} {d['unit']} ms={d['ms_per_step']:.4f} "
              f"kernel_ms={r.get('kernel_ms', 0):.4f} frac={r.get('frac', 0):.3f} "
              f"e2e={(d.get('e2e') or {}).get('value', 0):.1f}")
