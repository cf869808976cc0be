#!/bin/bash
# 1-GPU: GPU tests, then the bench under the pass-kernel loop variants (one line each)
O=gpurun_out
P=${1:-t3}
timeout 1200 python -m pytest tests -m gpu -x -q -k "not sharded" > $O/${P}_pytest.log 2>&1; tail -1 $O/${P}_pytest.log
for cfg in "" "SVB200_JIT_PP=1" "SVB200_JIT_PP=1 SVB200_JIT_PP_FREE=1" "SVB200_JIT_SPLIT=1" "SVB200_TAN=0" "SVB200_JIT_CTAS=3"; do
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
