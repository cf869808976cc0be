#!/bin/bash
# 2-GPU scale/parity session (round 2): parity at 30/33 qubits, sharded timings
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1"
O=gpurun_out
export SVB200_NCCL_TIMEOUT=300
timeout 600 $TR --master-port 29501 benchmarks/scale_parity.py --check agree --qubits 30 --depth 10 > $O/s2_agree30.jsonl 2> $O/s2_agree30.err
timeout 600 $TR --master-port 29502 benchmarks/scale_parity.py --check qaoa --qubits 33 --adjoint > $O/s2_qaoa33.jsonl 2> $O/s2_qaoa33.err
timeout 600 $TR --master-port 29503 benchmarks/adjoint_bench.py --config 3 --qubits 33 --skip-unfused > $O/s2_adj33_p2.jsonl 2> $O/s2_adj33_p2.err
timeout 600 $TR --master-port 29504 bench.py --gpus 2 --steps 5 --warmup 3 > $O/s2_bench31.json 2> $O/s2_bench31.err
timeout 900 $TR --master-port 29505 bench.py --gpus 2 --n-qubits 34 --steps 3 --warmup 2 --cpu-seconds 2 > $O/s2_bench34.json 2> $O/s2_bench34.err
for f in $O/s2_*.json*; do echo "== $f"; tail -c 600 $f; echo; done
