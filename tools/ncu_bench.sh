#!/bin/bash
# Launch list of the timed steps + one full capture of a kernel (run under gpurun, 1 GPU).
#   tools/ncu_bench.sh <tag> <kernel-regex> [bench args...]
tag=$1; kre=$2; shift 2
export BENCH_NVTX=1
timeout 900 ncu --nvtx --nvtx-include "timed/" --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/ncu_list_${tag}.log 2>&1
timeout 900 ncu --nvtx --nvtx-include "timed/" --set full --clock-control none --import-source on -k regex:"${kre}" -c 8 \
  -o gpurun_out/prof_${tag} python bench.py --steps 2 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/ncu_full_${tag}.log 2>&1
ls gpurun_out
