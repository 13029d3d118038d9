"""One-line summary of a bench.py JSON line read from stdin."""
import json
import sys

lines = [l for l in sys.stdin.read().strip().splitlines() if l.startswith("{")]
if not lines:
    print("no JSON line")
    sys.exit(0)
d = json.loads(lines[-1])
e2e = (d.get("e2e") or {}).get("value")
print(d.get("value"), d.get("ms_per_step"), (d.get("roofline") or {}).get("frac"), d.get("clocks"), "e2e", e2e,
      (d.get("config") or {}).get("state"))
