mkdir -p gpurun_out
(for d in 0 1 2 4 7; do echo "== dbg $d"; SDV2_GEMM_DBG=$d SDV2_GEMM_CFG=2,224,0 timeout 60 python tools/gemm_trace.py 1560 8960 1536 1 | sed -n 2,6p; done
 for d in 0 1 4; do echo "== dbg $d"; SDV2_GEMM_DBG=$d SDV2_GEMM_CFG=1,160,0 timeout 60 python tools/gemm_trace.py 1560 1536 1536 0 | sed -n 2,3p; done
 for sh in "1560 512 12" "1560 7800 12"; do timeout 60 python tools/attn_cta.py $sh | tail -8; done
) > gpurun_out/c6.log 2>&1
cat gpurun_out/c6.log | tail -150
