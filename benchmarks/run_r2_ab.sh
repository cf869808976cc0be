#!/bin/bash
# 1-GPU A/B of planner / kernel knobs on the bench circuit: "cfg1;cfg2;..." alternating, twice
O=gpurun_out
P=${1:-ab}
IFS=';' read -ra CFGS <<< "${2:-;SVB200_PHASE_SEARCH=0}"
for rep in 1 2; do
for cfg in "${CFGS[@]}"; do
  env $cfg timeout 600 python bench.py --steps 5 --warmup 3 --no-adjoint --cpu-seconds 1 > $O/${P}_sweep.tmp 2> $O/${P}_sweep.err
  python - "$cfg" $O/${P}_sweep.tmp >> $O/${P}_sweep.txt <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"[{sys.argv[1]}] s/circuit {d['s_per_circuit']:.4f} frac {d['roofline']['frac']:.3f} launches {d['roofline']['launches']} clocks {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
except Exception as e:
    print(f"[{sys.argv[1]}] failed: {e}")
PY
done
done
cat $O/${P}_sweep.txt
