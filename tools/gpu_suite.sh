#!/bin/bash
# GPU suite + default bench: tools/gpu_suite.sh <tag>
tag=${1:-x}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_${tag}.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_${tag}.log
timeout 400 python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
tail -3 gpurun_out/pytest_gpu_${tag}.log; cut -c1-400 gpurun_out/bench_${tag}.json
python -c "import json; d=json.load(open('gpurun_out/bench_${tag}.json')); print(d['roofline']['classes'], d['clocks'])"
