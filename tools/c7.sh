mkdir -p gpurun_out
(timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -3
 SDV2_GEMM_CFG=2,224,0 timeout 60 python tools/gemm_trace.py 1560 8960 1536 1 | sed -n 1,7p
 SDV2_GEMM_CFG=1,160,0 timeout 60 python tools/gemm_trace.py 1560 1536 1536 0 | sed -n 1,3p
 SDV2_GEMM_CFG=1,160,0 timeout 60 python tools/gemm_trace.py 1560 1536 1536 2 | sed -n 1,3p
 SDV2_VERBOSE=1 SDV2_PROF_DETAIL=1 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/b7.json 2> gpurun_out/b7.err; cut -c1-300 gpurun_out/b7.json; grep -v cand gpurun_out/b7.err | tail -20
) > gpurun_out/c7.log 2>&1
cat gpurun_out/c7.log | tail -150
