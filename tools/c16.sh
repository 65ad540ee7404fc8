mkdir -p gpurun_out
(timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
 SDV2_VERBOSE=1 timeout 300 python bench.py --no-cpu-baseline --steps 50 2>&1 >/dev/null | grep "gemm tune"
 bash tools/ab.sh wg2 main
 timeout 600 python bench.py --config long_horizon --steps 1000 --warmup 5 --no-cpu-baseline > gpurun_out/bench_long_r1g.json 2> gpurun_out/bench_long_r1g.err; cut -c1-400 gpurun_out/bench_long_r1g.json
) > gpurun_out/c16.log 2>&1
cat gpurun_out/c16.log | tail -40
