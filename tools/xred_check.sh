#!/bin/bash
# residual reduce-add epilogue: kernel tests, parity, A/B vs the x-tile read-modify-write build
mkdir -p gpurun_out
(timeout 400 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3
 timeout 120 python tools/time_gemm_sk.py 2>&1 | grep -v "^sdv2" | cut -c1-200
 bash tools/ab.sh main noxred
) > gpurun_out/xred.log 2>&1
cat gpurun_out/xred.log
