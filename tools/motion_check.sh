#!/bin/bash
mkdir -p gpurun_out
(timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_clean_rerun.py tests/test_gpu_pipeline.py -x -q 2>&1 | tail -2
 bash tools/ab.sh main head
) > gpurun_out/motion.log 2>&1
cat gpurun_out/motion.log
