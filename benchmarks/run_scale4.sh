#!/bin/bash
# 4-GPU scale/parity session (round 2): U.U^dagger round trips at 34/35 qubits, 34q adjoint, sharded timings
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
O=gpurun_out
export SVB200_NCCL_TIMEOUT=300
timeout 900 $TR --master-port 29511 benchmarks/scale_parity.py --check roundtrip --qubits 34 --depth 20 > $O/s4_rt34.jsonl 2> $O/s4_rt34.err
timeout 900 $TR --master-port 29512 benchmarks/scale_parity.py --check roundtrip --qubits 35 --depth 20 > $O/s4_rt35.jsonl 2> $O/s4_rt35.err
timeout 900 $TR --master-port 29513 benchmarks/scale_parity.py --check qaoa --qubits 34 --adjoint > $O/s4_qaoa34.jsonl 2> $O/s4_qaoa34.err
timeout 900 $TR --master-port 29514 benchmarks/adjoint_bench.py --config 3 --qubits 34 --skip-unfused > $O/s4_adj34.jsonl 2> $O/s4_adj34.err
timeout 600 $TR --master-port 29515 bench.py --gpus 4 --steps 5 --warmup 3 > $O/s4_bench32.json 2> $O/s4_bench32.err
timeout 900 $TR --master-port 29516 bench.py --gpus 4 --n-qubits 34 --steps 3 --warmup 2 --cpu-seconds 2 > $O/s4_bench34.json 2> $O/s4_bench34.err
timeout 900 $TR --master-port 29517 bench.py --gpus 4 --n-qubits 35 --steps 3 --warmup 2 --cpu-seconds 2 > $O/s4_bench35.json 2> $O/s4_bench35.err
for f in $O/s4_*.json*; do echo "== $f"; tail -c 700 $f; echo; done
