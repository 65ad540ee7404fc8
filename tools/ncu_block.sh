#!/bin/bash
# One full ncu capture of the 8 tensor-core launches of the first DiT block in the timed
# region (QKV, self-attn, O, cross-Q, cross-attn, cross-O, FFN1, FFN2).   tools/ncu_block.sh <tag>
tag=$1; shift
export BENCH_NVTX=1
timeout 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
  -k regex:"gemm_tc_kernel|attn_tc_kernel" -c 8 -o gpurun_out/block_${tag} \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/ncu_block_${tag}.log 2>&1
