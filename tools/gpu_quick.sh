# quick GPU check: kernel/gemm tests + GEMM and attention micro-benchmarks
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_gemm_gpu.py -q -x > gpurun_out/q_tests.log 2>&1; echo rc=$? >> gpurun_out/q_tests.log
timeout 600 python tools/gemm_bench.py --json gpurun_out/gemm_bench.json > gpurun_out/gemm_bench.log 2>&1; echo rc=$? >> gpurun_out/gemm_bench.log
DP_FA_EMU=${EMU:-2} timeout 300 python tools/attn_bench.py > gpurun_out/attn.log 2>&1
