#!/bin/bash
# round-2 end-of-work session on ONE B200: tests, smoke, bench, results rows, ncu launch list + one full capture
O=gpurun_out
P=${1:-f1}
timeout 1200 python -m pytest tests -m gpu -q > $O/${P}_pytest.log 2>&1; tail -2 $O/${P}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${P}_smoke.log 2>&1; tail -1 $O/${P}_smoke.log
timeout 900 python bench.py > $O/${P}_bench.json 2> $O/${P}_bench.err; python benchmarks/show_bench.py $O/${P}_bench.json | head -4
timeout 900 python benchmarks/results.py --rows 1,3,5 > $O/${P}_results.jsonl 2> $O/${P}_results.err; cat $O/${P}_results.jsonl | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${P}_launches.csv python bench.py --steps 2 --warmup 1 --no-adjoint --cpu-seconds 1 > $O/${P}_ncu_launch.log 2>&1; tail -1 $O/${P}_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:svb200_pass -s 40 -c 1 -o $O/${P}_pass40 python bench.py --steps 1 --warmup 3 --no-adjoint --cpu-seconds 1 > $O/${P}_ncu_full.log 2>&1; tail -1 $O/${P}_ncu_full.log
timeout 300 python bench.py --impl reference --steps 3 --warmup 3 > $O/${P}_ref.json 2> $O/${P}_ref.err; tail -c 400 $O/${P}_ref.json
