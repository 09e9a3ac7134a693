mkdir -p gpurun_out
timeout 900 python tools/conv_bench.py --json gpurun_out/conv_bench.json > gpurun_out/conv_bench.log 2>&1; echo rc=$? >> gpurun_out/conv_bench.log
DP_FA_EMU=${EMU:-2} timeout 300 python tools/attn_bench.py > gpurun_out/attn.log 2>&1
