mkdir -p gpurun_out
(timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
 SDV2_GEMM_CFG=2,224,0 timeout 60 python tools/gemm_trace.py 1560 8960 1536 1 | sed -n 2,6p
 SDV2_GEMM_CFG=2,224,0 timeout 60 python tools/gemm_cta.py 1560 8960 1536 1 | tail -1
 SDV2_GEMM_CFG=1,160,0 timeout 60 python tools/gemm_cta.py 1560 1536 1536 2 | tail -1
 timeout 120 python tools/time_gemm.py
 bash tools/ab.sh split2 main wg2 wg4
) > gpurun_out/c12.log 2>&1
cat gpurun_out/c12.log | tail -150
