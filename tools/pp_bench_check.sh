#!/bin/bash
# Pipeline bench logic with 2 ranks on ONE GPU (gloo host staging instead of NCCL).
SDV2_PP_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps ${1:-20} --warmup 3 ${2:+--config $2}
