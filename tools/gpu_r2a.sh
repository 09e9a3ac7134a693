mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
bash tools/gpu_tests.sh tests/test_kernels_gpu.py tests/test_gemm_gpu.py tests/test_c1_parity_gpu.py tests/test_c2_parity_gpu.py tests/test_ext_configs_gpu.py tests/test_cuda_graph_gpu.py tests/test_flip_cache_gpu.py tests/test_memory_gpu.py tests/test_optimizer_overlap_gpu.py tests/test_pipeline_multiproc_gpu.py tests/test_profiling_run_gpu.py tests/test_zz_bench_config_parity_gpu.py
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$? >> gpurun_out/bench.log
