#!/bin/bash
# One full ncu capture of every launch of the first DiT block in the timed region (norm1,
# QKV, qkv_post, self-attn, O, norm3, cross-Q, q RMS, cross-attn, cross-O, norm2, FFN1,
# FFN2) plus the launch list of the whole timed region.   tools/ncu_block.sh <tag> [bench args]
tag=$1; shift
export BENCH_NVTX=1
mkdir -p gpurun_out
# the GEMM configurations are tuned once without the profiler (under ncu every timed
# candidate is a cold serialised launch) and pinned for the profiled runs
table=gpurun_out/gemm_table_${tag}.json
rm -f $table
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --latency-chunks 0 --gemm-table $table "$@" \
  > gpurun_out/bench_pre_${tag}.json 2> gpurun_out/bench_pre_${tag}.err
set -- --gemm-table $table "$@"
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --latency-chunks 0 "$@" \
  > gpurun_out/ncu_list_${tag}.log 2>&1
timeout 1200 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on \
  -k regex:"gemm_tc_kernel|attn_tc_kernel|xattn_tc_kernel|norm_mod2|qkv_post2|rms_rows2" -c 13 -o gpurun_out/block_${tag} \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --latency-chunks 0 "$@" > gpurun_out/ncu_block_${tag}.log 2>&1
ls -la gpurun_out | grep ${tag}
