mkdir -p gpurun_out
(bash tools/time_attn_ab.sh main poly0x00 poly0x44 poly0xAA
 bash tools/ab.sh main poly0x44 poly0xAA
) > gpurun_out/c17.log 2>&1
cat gpurun_out/c17.log | tail -40
