mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_profiling_run_gpu.py -q -x -k "two_ranks" > gpurun_out/prof_test.log 2>&1; echo rc=$? >> gpurun_out/prof_test.log
timeout 600 python tools/gemm_bench.py --only dgrad --json gpurun_out/gemm_dgrad.json > gpurun_out/gemm_dgrad.log 2>&1
timeout 600 python tools/host_profile.py > gpurun_out/host_profile.log 2>&1
