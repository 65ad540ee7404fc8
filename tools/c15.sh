mkdir -p gpurun_out
(echo "== reset test on the previous build (expected to fail)"; SDV2_LIB_PATH=$PWD/paper_2511_07399_b200/variants/libsdv2_wg2.so timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "reset_with_new" 2>&1 | tail -2
 bash tools/ncu_block.sh r1g
 python tools/ncu_traffic.py gpurun_out/block_r1g.ncu-rep gpurun_out/r1g_ncu_traffic.json wan13_480p_1step
 timeout 300 python bench.py --steps 100 > gpurun_out/bench_r1g.json 2> gpurun_out/bench_r1g.err; cut -c1-300 gpurun_out/bench_r1g.json
) > gpurun_out/c15.log 2>&1
cat gpurun_out/c15.log | tail -50
