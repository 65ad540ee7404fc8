(bash tools/ab.sh base packed db; timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2) > gpurun_out/c8.log 2>&1; cat gpurun_out/c8.log
