mkdir -p gpurun_out
(bash tools/pp_bench_check.sh 20 > gpurun_out/pp2.json 2> gpurun_out/pp2.err; echo "pp exit $?"; cut -c1-3000 gpurun_out/pp2.json; tail -5 gpurun_out/pp2.err
 timeout 120 python tools/time_gemm.py
 EPIS=0 timeout 60 python tools/time_attn.py
 timeout 60 python tools/gemm_trace.py 1560 1536 1536 2
 timeout 60 python tools/gemm_trace.py 1560 1536 1536 0
) > gpurun_out/c2.log 2>&1
cat gpurun_out/c2.log | tail -150
