#!/bin/bash
# 1-GPU: GPU tests with the DFL pass loop, then the bench alternating default / DFL
O=gpurun_out
P=${1:-t4}
SVB200_JIT_DFL=1 timeout 1200 python -m pytest tests -m gpu -x -q -k "not sharded" > $O/${P}_pytest_dfl.log 2>&1; tail -1 $O/${P}_pytest_dfl.log
for cfg in "" "SVB200_JIT_DFL=1" "" "SVB200_JIT_DFL=1" "SVB200_JIT_DFL=1 SVB200_JIT_CTAS=3"; do
  env $cfg timeout 600 python bench.py --steps 5 --warmup 3 --no-adjoint --cpu-seconds 1 > $O/${P}_sweep.tmp 2> $O/${P}_sweep.err
  python - "$cfg" $O/${P}_sweep.tmp >> $O/${P}_sweep.txt <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    print(f"[{sys.argv[1]}] s/circuit {d['s_per_circuit']:.4f} frac {d['roofline']['frac']:.3f} clocks {d['clocks']['sm_mhz']} {d['clocks']['reasons']}")
except Exception as e:
    print(f"[{sys.argv[1]}] failed: {e}")
PY
done
cat $O/${P}_sweep.txt
SVB200_JIT_DFL=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:svb200_pass -s 40 -c 1 -o $O/${P}_ncu_pass_dfl \
  python bench.py --steps 1 --warmup 3 --no-adjoint --cpu-seconds 1 > $O/${P}_ncu_full.log 2>&1; tail -1 $O/${P}_ncu_full.log
