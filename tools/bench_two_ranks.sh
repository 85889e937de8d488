#!/bin/bash
# Two bench ranks on ONE GPU (gloo collectives): exercises the N > 1 code paths of bench.py where
# only one GPU is available.  The numbers are meaningless (the ranks share the device).
W=${1:-c4_xyz_14_2}
for mode in strong weak; do
  QX_BENCH_BACKEND=gloo QX_BENCH_SHARE_GPU=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
      --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 2 --warmup 1 --workload $W --scaling $mode --no-cpu
done
python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29518 \
    bench.py --gpus 2 --steps 1 --warmup 0 --workload c4_xyz_12_2 --impl reference
