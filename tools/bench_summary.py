import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["clocks"], d["e2e"]["value"], d["config"].get("state"))
