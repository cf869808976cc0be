#!/bin/bash
# 1-GPU session: tests touched this round, per-gate sweeps, ncu of k_pair, sanitizer runs
O=gpurun_out
timeout 900 python -m pytest tests/test_batching.py tests/test_gpu_parity.py tests/test_gpu_f32.py -q -x > $O/r2s_pytest.log 2>&1; tail -1 $O/r2s_pytest.log
timeout 600 python benchmarks/results.py --rows 2,2c > $O/r2s_results.jsonl 2> $O/r2s_results.err; tail -c 1500 $O/r2s_results.jsonl
cat > /tmp/rx30.py <<'PY'
import sys; sys.path.insert(0, ".")
from paper_2403_02512_b200.device import Device
from paper_2403_02512_b200.ops import Op
with Device(30, fuse=False) as d:
    for _ in range(3):
        d.apply([Op("RX", (15,), (0.3,))])
    d.synchronize()
PY
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pair -s 1 -c 1 -o $O/r2_ncu_kpair_rx30 python /tmp/rx30.py > $O/r2_ncu_kpair.log 2>&1; tail -2 $O/r2_ncu_kpair.log
for tool in racecheck synccheck memcheck; do
  SAN_N=13 timeout 900 compute-sanitizer --tool $tool --print-limit 20 python benchmarks/sanitize_fused.py > $O/r2_san_${tool}.log 2>&1; tail -3 $O/r2_san_${tool}.log
done
SVB200_JIT_PP=1 SAN_N=13 timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python benchmarks/sanitize_fused.py > $O/r2_san_racecheck_pp.log 2>&1; tail -3 $O/r2_san_racecheck_pp.log
