#!/bin/bash
# round-2 end-of-work session on TWO B200s: sharded + batching tests, N=2 bench lines, scale parity
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
O=gpurun_out
P=${1:-g2}
export SVB200_NCCL_TIMEOUT=300
timeout 1500 python -m pytest tests/test_gpu_sharded.py tests/test_batching.py -m gpu -q > $O/${P}_pytest.log 2>&1; tail -1 $O/${P}_pytest.log
timeout 600 $TR --master-port 29701 bench.py --gpus 2 --steps 5 --warmup 3 > $O/${P}_bench31.json 2> $O/${P}_bench31.err
timeout 900 $TR --master-port 29702 bench.py --gpus 2 --n-qubits 34 --steps 3 --warmup 2 --cpu-seconds 2 --no-adjoint > $O/${P}_bench34.json 2> $O/${P}_bench34.err
timeout 600 $TR --master-port 29703 benchmarks/scale_parity.py --check agree --qubits 30 --depth 10 > $O/${P}_agree30.jsonl 2> $O/${P}_agree30.err
timeout 600 $TR --master-port 29704 benchmarks/scale_parity.py --check qaoa --qubits 33 --adjoint > $O/${P}_qaoa33.jsonl 2> $O/${P}_qaoa33.err
timeout 600 $TR --master-port 29705 benchmarks/adjoint_bench.py --config 3 --qubits 33 --skip-unfused > $O/${P}_adj33.jsonl 2> $O/${P}_adj33.err
timeout 600 $TR --master-port 29706 benchmarks/exchange_bw.py --qubits 32 > $O/${P}_xchg32.jsonl 2> $O/${P}_xchg32.err
python benchmarks/show_bench.py $O/${P}_bench31.json $O/${P}_bench34.json | grep "==\|s_per_circuit\|comm\|adjoint"
for f in $O/${P}_agree30.jsonl $O/${P}_qaoa33.jsonl $O/${P}_adj33.jsonl $O/${P}_xchg32.jsonl; do grep -h "^{" $f | cut -c1-400; done
