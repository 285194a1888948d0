#!/bin/bash
# round-2 GPU pass bh: the N > 1 code path of bench.py (NCCL init, closing all-reduce / gather on the pipeline
# stream, barriers) with one rank under torchrun (VFPI_BENCH_FORCE_DIST=1), and the self-spawning --gpus 1 launch
cd $GRAFT_REPO_ROOT
export PYTHONUNBUFFERED=1
mkdir -p gpurun_out
VFPI_BENCH_FORCE_DIST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 1 --steps 2 --warmup 1 --no-cpu-baseline --no-subrecords > gpurun_out/r2bh_dist.json 2> gpurun_out/r2bh_dist.err; echo "rc $?"
tail -c 400 gpurun_out/r2bh_dist.json; tail -n 5 gpurun_out/r2bh_dist.err
