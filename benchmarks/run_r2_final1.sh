#!/bin/bash
# round-2 end-of-work session on ONE B200: tests, smoke, bench, results rows, ncu launch list + one full capture
O=gpurun_out
timeout 1200 python -m pytest tests -m gpu -q > $O/f1_pytest.log 2>&1; tail -2 $O/f1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/f1_smoke.log 2>&1; tail -1 $O/f1_smoke.log
timeout 900 python bench.py > $O/f1_bench.json 2> $O/f1_bench.err; python benchmarks/show_bench.py $O/f1_bench.json | head -4
timeout 900 python benchmarks/results.py --rows 1,3,5 > $O/f1_results.jsonl 2> $O/f1_results.err; cat $O/f1_results.jsonl | cut -c1-300
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/f1_launches.csv python bench.py --steps 2 --warmup 1 --no-adjoint --cpu-seconds 1 > $O/f1_ncu_launch.log 2>&1; tail -1 $O/f1_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:svb200_pass -s 40 -c 1 -o $O/f1_pass40 python bench.py --steps 1 --warmup 3 --no-adjoint --cpu-seconds 1 > $O/f1_ncu_full.log 2>&1; tail -1 $O/f1_ncu_full.log
