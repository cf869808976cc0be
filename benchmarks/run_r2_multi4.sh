#!/bin/bash
# round-2 end-of-work session on FOUR B200s: sharded tests at world 4, N=4 bench lines, 34/35q parity and adjoint
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
O=gpurun_out
P=${1:-g4}
export SVB200_NCCL_TIMEOUT=300
timeout 1200 python -m pytest tests/test_gpu_sharded.py -m gpu -q -k "not dead" > $O/${P}_pytest.log 2>&1; tail -1 $O/${P}_pytest.log
timeout 600 $TR --master-port 29801 bench.py --gpus 4 --steps 5 --warmup 3 > $O/${P}_bench32.json 2> $O/${P}_bench32.err
timeout 900 $TR --master-port 29802 bench.py --gpus 4 --n-qubits 34 --steps 3 --warmup 2 --cpu-seconds 2 --no-adjoint > $O/${P}_bench34.json 2> $O/${P}_bench34.err
timeout 900 $TR --master-port 29803 bench.py --gpus 4 --n-qubits 35 --steps 3 --warmup 2 --cpu-seconds 2 --no-adjoint > $O/${P}_bench35.json 2> $O/${P}_bench35.err
timeout 900 $TR --master-port 29804 benchmarks/scale_parity.py --check roundtrip --qubits 34 --depth 20 > $O/${P}_rt34.jsonl 2> $O/${P}_rt34.err
timeout 900 $TR --master-port 29805 benchmarks/scale_parity.py --check roundtrip --qubits 35 --depth 20 > $O/${P}_rt35.jsonl 2> $O/${P}_rt35.err
timeout 900 $TR --master-port 29806 benchmarks/scale_parity.py --check qaoa --qubits 34 --adjoint > $O/${P}_qaoa34.jsonl 2> $O/${P}_qaoa34.err
timeout 900 $TR --master-port 29807 benchmarks/adjoint_bench.py --config 3 --qubits 34 --skip-unfused > $O/${P}_adj34.jsonl 2> $O/${P}_adj34.err
timeout 600 $TR --master-port 29808 benchmarks/exchange_bw.py --qubits 33 > $O/${P}_xchg33.jsonl 2> $O/${P}_xchg33.err
python benchmarks/show_bench.py $O/${P}_bench32.json $O/${P}_bench34.json $O/${P}_bench35.json | grep "==\|s_per_circuit\|comm\|adjoint"
for f in $O/${P}_rt34.jsonl $O/${P}_rt35.jsonl $O/${P}_qaoa34.jsonl $O/${P}_adj34.jsonl $O/${P}_xchg33.jsonl; do grep -h "^{" $f | cut -c1-400; done
