mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/q_tests.log 2>&1; echo rc=$? >> gpurun_out/q_tests.log
timeout 900 python tools/conv_bench.py --no-cudnn --json gpurun_out/conv_bench4.json > gpurun_out/conv_bench4.log 2>&1
timeout 600 python tools/gemm_bench.py --json gpurun_out/gemm_bench4.json > gpurun_out/gemm_bench4.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1
