mkdir -p gpurun_out
(timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -40) > gpurun_out/c9b.log 2>&1
bash tools/c9.sh > /dev/null 2>&1
cat gpurun_out/c9b.log; cat gpurun_out/c9.log
