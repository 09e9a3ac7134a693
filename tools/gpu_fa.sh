mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "flash or attn" > gpurun_out/fa_tests.log 2>&1; echo rc=$? >> gpurun_out/fa_tests.log
DP_FA_EMU=${EMU:-2} timeout 300 python tools/attn_bench.py > gpurun_out/attn.log 2>&1
