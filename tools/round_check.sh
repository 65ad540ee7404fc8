#!/bin/bash
# Full round check on one B200: GPU suite, default bench (+cpu baseline), reference arm,
# the other configs, the SLO batch and serving loop, the Stream-VAE timing.
#   tools/round_check.sh <tag>
tag=${1:-r2z}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu_${tag}.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${tag}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${tag}.log
timeout 400 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${tag}.json 2> gpurun_out/bench_ref_${tag}.err
for c in wan13_512_4step wan14_480p_4step; do
  timeout 900 python bench.py --config $c --steps 20 --no-cpu-baseline --latency-chunks 256 > gpurun_out/bench_${c}_${tag}.json 2> gpurun_out/bench_${c}_${tag}.err
done
timeout 400 python bench.py --streams 4 --no-cpu-baseline --latency-chunks 256 > gpurun_out/bench_streams4_${tag}.json 2> gpurun_out/bench_streams4_${tag}.err
timeout 400 python bench.py --kv-mode clean --no-cpu-baseline --latency-chunks 256 > gpurun_out/bench_clean_${tag}.json 2> gpurun_out/bench_clean_${tag}.err
timeout 600 python -u tools/slo_serve.py gpurun_out/slo_serve_${tag}.json 100 80 6 > gpurun_out/slo_serve_${tag}.log 2>&1
timeout 300 python -u tools/vae_bench.py gpurun_out/vae_bench_${tag}.json > gpurun_out/vae_bench_${tag}.log 2>&1
tail -3 gpurun_out/pytest_gpu_${tag}.log; for f in gpurun_out/bench*_${tag}.json; do echo $f; cut -c1-300 $f; done; tail -1 gpurun_out/slo_serve_${tag}.log | cut -c1-600
