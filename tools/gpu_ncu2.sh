mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 2 -c 1 -o gpurun_out/gemm_fwd_1280b python tools/gemm_one.py 2048 1280 1280 fwd 4 > gpurun_out/ncu9.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fa_fwd -s 1 -c 1 -o gpurun_out/fa_fwd2 python tools/attn_bench.py > gpurun_out/ncu10.log 2>&1
