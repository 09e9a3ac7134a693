mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_kernels_gpu.py -q -x > gpurun_out/k_tests.log 2>&1; echo rc=$? >> gpurun_out/k_tests.log
timeout 600 python -m pytest tests/test_c2_parity_gpu.py tests/test_ext_configs_gpu.py tests/test_flip_cache_gpu.py tests/test_optimizer_overlap_gpu.py -q -x > gpurun_out/geglu_parity.log 2>&1; echo rc=$? >> gpurun_out/geglu_parity.log
timeout 500 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
