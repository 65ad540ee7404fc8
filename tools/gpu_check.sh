mkdir -p gpurun_out
(timeout 200 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -3
 timeout 90 python tools/time_attn.py
 SDV2_ATTN_PER_UNIT=1 timeout 90 python tools/time_attn.py
 timeout 120 python tools/time_gemm.py
 timeout 400 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_elect.json 2> gpurun_out/bench_elect.err; cat gpurun_out/bench_elect.json | cut -c1-400
) > gpurun_out/elect.log 2>&1
cat gpurun_out/elect.log
