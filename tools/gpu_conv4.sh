mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/q_tests.log 2>&1; echo rc=$? >> gpurun_out/q_tests.log
timeout 900 python tools/conv_bench.py --no-cudnn --json gpurun_out/conv_bench3.json > gpurun_out/conv_bench3.log 2>&1
timeout 600 python tools/gemm_bench.py --json gpurun_out/gemm_bench3.json > gpurun_out/gemm_bench3.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv >> gpurun_out/q_tests.log
