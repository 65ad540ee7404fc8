mkdir -p gpurun_out
(bash tools/pp_bench_check.sh 20 > gpurun_out/pp2.json 2> gpurun_out/pp2.err; echo "pp exit $?"; cut -c1-3000 gpurun_out/pp2.json; grep -v "^\s*$" gpurun_out/pp2.err | tail -5
 SDV2_VERBOSE=2 SDV2_PROF_DETAIL=1 timeout 300 python bench.py --no-cpu-baseline --steps 50 > gpurun_out/b3.json 2> gpurun_out/b3.err; cut -c1-400 gpurun_out/b3.json; grep -v cand gpurun_out/b3.err | tail -40
 timeout 60 python tools/attn_trace.py 1560 512 12
) > gpurun_out/c3.log 2>&1
cat gpurun_out/c3.log | tail -150
