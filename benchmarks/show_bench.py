"""Print the headline keys of bench.py JSON lines (files given on the command line)."""
import json
import sys

for path in sys.argv[1:]:
    lines = [x for x in open(path).read().splitlines() if x.startswith("{")]
    if not lines:
        print(path, "no JSON line")
        continue
    d = json.loads(lines[-1])
    print("==", path)
    for k in ("s_per_circuit", "value", "e2e", "e2e_cold", "e2e_repeat", "adjoint", "clocks", "comm", "gpu_launches"):
        if k in d:
            print(f"  {k}: {d[k]}")
    if "roofline" in d:
        r = d["roofline"]
        print(f"  roofline frac {r.get('frac')} fp64 {r.get('fp64', {}).get('frac')}")
