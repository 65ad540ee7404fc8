mkdir -p gpurun_out
(timeout 300 python -m pytest tests/test_gpu_kernels.py -x -q -k "attn or attention" 2>&1 | tail -3
 timeout 90 python tools/time_attn.py
 for sh in "1560 512 12" "1560 7800 12"; do timeout 60 python tools/attn_cta.py $sh | tail -8; done
 SDV2_LIB_PATH=$PWD/paper_2511_07399_b200/variants/libsdv2_split2.so timeout 90 python tools/time_attn.py
 bash tools/ab.sh split2 main
) > gpurun_out/c11.log 2>&1
cat gpurun_out/c11.log | tail -150
