#!/bin/bash
# sanitizers on the tiny stream (+ clean re-run, GEMM / attention hooks) and the 10k-chunk long horizon
tag=${1:-r2zd}
mkdir -p gpurun_out
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_tiny.py > gpurun_out/san_memcheck_${tag}.log 2>&1; echo "memcheck exit $?" >> gpurun_out/san_memcheck_${tag}.log
timeout 1800 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_tiny.py > gpurun_out/san_racecheck_${tag}.log 2>&1; echo "racecheck exit $?" >> gpurun_out/san_racecheck_${tag}.log
timeout 1500 python -u tools/long_horizon.py gpurun_out/long_horizon_10k_${tag}.json 10000 > gpurun_out/long_horizon_${tag}.log 2>&1; echo "long horizon exit $?" >> gpurun_out/long_horizon_${tag}.log
tail -4 gpurun_out/san_memcheck_${tag}.log; tail -4 gpurun_out/san_racecheck_${tag}.log; tail -3 gpurun_out/long_horizon_${tag}.log
