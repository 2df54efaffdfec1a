"""Summarise a bench.py JSON line from stdin: tag, ms/step, value, per-class (ms, frac)."""
import json, sys
tag = sys.argv[1] if len(sys.argv) > 1 else ""
lines = [l for l in sys.stdin.read().strip().splitlines() if l.startswith("{")]
if not lines:
    print(tag, "NO JSON")
    sys.exit(0)
d = json.loads(lines[-1])
pc = d.get("roofline", {}).get("per_class", {})
print(tag, round(d["ms_per_step"], 3), round(d["value"], 1),
      {k: (round(v["ms_per_step"], 2), round(v.get("frac", 0), 3)) for k, v in pc.items()})
