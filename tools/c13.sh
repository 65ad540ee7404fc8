mkdir -p gpurun_out
(timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q 2>&1 | tail -2
 timeout 90 python tools/time_attn.py
 for sh in "1560 512 12"; do timeout 60 python tools/attn_cta.py $sh | tail -8; done
 bash tools/ab.sh wg2 main
) > gpurun_out/c13.log 2>&1
cat gpurun_out/c13.log | tail -150
