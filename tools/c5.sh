mkdir -p gpurun_out
(SDV2_GEMM_CFG=2,224,0 timeout 60 python tools/gemm_trace.py 1560 8960 1536 1
 SDV2_GEMM_CFG=1,224,0 timeout 60 python tools/gemm_trace.py 1560 8960 1536 1
 SDV2_GEMM_CFG=2,160,0 timeout 60 python tools/gemm_trace.py 1560 1536 8960 2
 for c in 1,256,0 2,256,0 1,224,0 2,224,0 1,192,0 2,192,0 2,128,0; do SDV2_GEMM_CFG=$c timeout 60 python tools/gemm_cta.py 1560 8960 1536 1 | tail -6; done
) > gpurun_out/c5.log 2>&1
cat gpurun_out/c5.log | tail -150
