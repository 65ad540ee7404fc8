#!/bin/bash
# Round-2 measurement batch (one B200): sanitizers, E10 stream batch on/off, W sweep,
# the 10k-chunk long-horizon run.   bash tools/r2_measure.sh <tag>
tag=${1:-r2f}
mkdir -p gpurun_out
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --error-exitcode 99 python tools/sanitize_tiny.py > gpurun_out/san_${t}_${tag}.log 2>&1
  echo "sanitizer $t exit $?" >> gpurun_out/san_${t}_${tag}.log
  tail -3 gpurun_out/san_${t}_${tag}.log
done
timeout 400 python bench.py --config wan13_512_4step --no-cpu-baseline --steps 60 --latency-chunks 0 > gpurun_out/e10_on_${tag}.json 2> gpurun_out/e10_on_${tag}.err
timeout 400 python bench.py --config wan13_512_4step --denoise-steps 1 --no-cpu-baseline --steps 120 --latency-chunks 0 > gpurun_out/e10_off_${tag}.json 2> gpurun_out/e10_off_${tag}.err
python tools/stream_batch.py gpurun_out/e10_${tag}.json gpurun_out/e10_on_${tag}.json gpurun_out/e10_off_${tag}.json
for w in 2 8; do
  timeout 400 python bench.py --config wan13_512_4step --window $w --no-cpu-baseline --steps 60 --latency-chunks 0 > gpurun_out/wsweep_W${w}_${tag}.json 2> gpurun_out/wsweep_W${w}_${tag}.err
  cut -c1-200 gpurun_out/wsweep_W${w}_${tag}.json
done
timeout 1200 python tools/long_horizon.py gpurun_out/long_horizon_${tag}.json > gpurun_out/long_horizon_${tag}.log 2>&1
tail -2 gpurun_out/long_horizon_${tag}.log
