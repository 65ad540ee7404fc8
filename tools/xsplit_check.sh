#!/bin/bash
mkdir -p gpurun_out
(timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k attention 2>&1 | tail -3
 timeout 60 python tools/time_attn.py 2>&1 | head -2
 timeout 400 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
 bash tools/ab.sh main noxsplit
) > gpurun_out/xsplit.log 2>&1
cat gpurun_out/xsplit.log
