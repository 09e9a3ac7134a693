mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -k "geglu or flip_batch" > gpurun_out/geglu_tests.log 2>&1; echo rc=$? >> gpurun_out/geglu_tests.log
