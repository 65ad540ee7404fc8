#!/bin/bash
# Full round check on one B200: GPU suite, default bench (+cpu baseline), reference arm,
# other configs, ncu launch list + full capture of the top kernels.
#   tools/round_check.sh <tag>
tag=${1:-r1e}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_${tag}.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${tag}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${tag}.log
timeout 400 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${tag}.json 2> gpurun_out/bench_ref_${tag}.err
for c in wan13_512_4step wan14_480p_4step; do
  timeout 600 python bench.py --config $c --steps 20 --no-cpu-baseline > gpurun_out/bench_${c}_${tag}.json 2> gpurun_out/bench_${c}_${tag}.err
done
bash tools/ncu_bench.sh ${tag} "gemm_tc|attn_tc|qkv_post|norm_mod"
bash tools/pp_bench_check.sh 30 > gpurun_out/pp2_${tag}.json 2> gpurun_out/pp2_${tag}.err
tail -3 gpurun_out/pytest_gpu_${tag}.log; cut -c1-600 gpurun_out/bench_${tag}.json; cut -c1-300 gpurun_out/bench_*_${tag}.json
