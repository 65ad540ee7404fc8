mkdir -p gpurun_out
(timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "reset_with_new" 2>&1 | tail -3
 timeout 300 python bench.py --no-cpu-baseline --steps 100 | cut -c1-200 ; 
 timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
) > gpurun_out/c14.log 2>&1
cat gpurun_out/c14.log | tail -50
