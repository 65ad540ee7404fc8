#!/bin/bash
mkdir -p gpurun_out
(timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q 2>&1 | tail -2
 bash tools/ab.sh main head
) > gpurun_out/gemv.log 2>&1
cat gpurun_out/gemv.log
