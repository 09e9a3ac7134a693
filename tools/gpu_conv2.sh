mkdir -p gpurun_out
DP_FORCE_CG=2 timeout 900 python tools/conv_bench.py --no-cudnn --json gpurun_out/conv_bench_cg2.json > gpurun_out/conv_bench_cg2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/wgrad_16_640 python tools/conv_one.py 32 16 16 640 640 1 wgrad 2 > gpurun_out/ncu5.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 1 -c 1 -o gpurun_out/wgrad_32_320 python tools/conv_one.py 32 32 32 320 320 1 wgrad 2 > gpurun_out/ncu6.log 2>&1
