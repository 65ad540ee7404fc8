mkdir -p gpurun_out
(for sh in "1560 512 12" "1560 7800 12" "1560 1560 12"; do timeout 60 python tools/attn_cta.py $sh; done
 SDV2_GEMM_CFG=1,160,0 timeout 60 python tools/gemm_cta.py 1560 1536 1536 2
 SDV2_GEMM_CFG=1,160,0 timeout 60 python tools/gemm_cta.py 1560 1536 1536 0
 SDV2_GEMM_CFG=2,224,0 timeout 60 python tools/gemm_cta.py 1560 8960 1536 1
 SDV2_GEMM_CFG=1,160,0 timeout 60 python tools/gemm_trace.py 1560 1536 1536 0
) > gpurun_out/c4.log 2>&1
cat gpurun_out/c4.log | tail -150
