mkdir -p gpurun_out
(for d in 0 8; do echo "== dbg $d"; SDV2_GEMM_DBG=$d SDV2_GEMM_CFG=2,224,0 timeout 60 python tools/gemm_trace.py 1560 8960 1536 1 | sed -n 2,6p; SDV2_GEMM_DBG=$d SDV2_GEMM_CFG=2,224,0 timeout 60 python tools/gemm_cta.py 1560 8960 1536 1 | tail -1; SDV2_GEMM_DBG=$d SDV2_GEMM_CFG=1,160,0 timeout 60 python tools/gemm_cta.py 1560 1536 1536 0 | tail -1; done
) > gpurun_out/c9.log 2>&1
cat gpurun_out/c9.log | tail -150
