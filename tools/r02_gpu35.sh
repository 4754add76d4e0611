#!/bin/bash
# smoke(), and the bench under torchrun at N=1 (the driver's launch form)
cd "$(dirname "$0")/.."
o=gpurun_out/r02ag
mkdir -p $o
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1; echo "smoke rc=$?"; tail -5 $o/smoke.txt
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 3 --warmup 3 > $o/bench_torchrun.json 2> $o/bench_torchrun.err; echo "torchrun rc=$?"; tail -c 400 $o/bench_torchrun.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 1 --steps 2 --warmup 3 > $o/ref_torchrun.json 2> $o/ref_torchrun.err; echo "ref torchrun rc=$?"; tail -c 300 $o/ref_torchrun.json
