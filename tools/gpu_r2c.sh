mkdir -p gpurun_out
python -m pytest tests/test_kernels_gpu.py -q -x -k "flash or attn" > gpurun_out/fa_tests.log 2>&1; echo rc=$? >> gpurun_out/fa_tests.log
for e in 0 2 4 8; do echo "EMU=$e" >> gpurun_out/attn.log; DP_FA_EMU=$e timeout 300 python tools/attn_bench.py >> gpurun_out/attn.log 2>&1; done
timeout 600 python tools/gemm_bench.py --json gpurun_out/gemm_bench.json > gpurun_out/gemm_bench.log 2>&1; echo rc=$? >> gpurun_out/gemm_bench.log
