#!/bin/bash
# 1-GPU session after the scaled-rotation (TAN/COT) change: GPU tests, bench, ncu launch list + one full capture
O=gpurun_out
P=${1:-t2}
timeout 1200 python -m pytest tests -m gpu -x -q -k "not sharded" > $O/${P}_pytest.log 2>&1; tail -1 $O/${P}_pytest.log
timeout 600 python bench.py > $O/${P}_bench.json 2> $O/${P}_bench.err; tail -c 600 $O/${P}_bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${P}_launches.csv \
  python bench.py --steps 2 --warmup 1 --no-adjoint --cpu-seconds 1 > $O/${P}_ncu_launches.log 2>&1; tail -1 $O/${P}_ncu_launches.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:svb200_pass -s 40 -c 1 -o $O/${P}_ncu_pass \
  python bench.py --steps 1 --warmup 3 --no-adjoint --cpu-seconds 1 > $O/${P}_ncu_full.log 2>&1; tail -1 $O/${P}_ncu_full.log
