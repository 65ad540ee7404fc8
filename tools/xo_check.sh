#!/bin/bash
mkdir -p gpurun_out
(timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k attention 2>&1 | tail -2
 timeout 100 python tools/xattn_cta.py 2>&1 | tail -10
 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_clean_rerun.py -x -q 2>&1 | tail -2
 bash tools/ab.sh main head
) > gpurun_out/xo.log 2>&1
cat gpurun_out/xo.log
