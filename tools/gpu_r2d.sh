mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/gemm_fwd_2560 python tools/gemm_one.py 32768 2560 320 fwd 2 > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/gemm_wgrad_1280 python tools/gemm_one.py 2048 1280 1280 wgrad 2 > gpurun_out/ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/gemm_fwd_1280 python tools/gemm_one.py 2048 1280 1280 fwd 2 > gpurun_out/ncu3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fa_fwd -s 1 -c 1 -o gpurun_out/fa_fwd python tools/attn_bench.py > gpurun_out/ncu4.log 2>&1
