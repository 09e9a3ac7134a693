mkdir -p gpurun_out
timeout -s KILL 2000 python -m pytest tests/test_zz_bench_config_parity_gpu.py -q -x -s > gpurun_out/bcp.log 2>&1; echo rc=$? >> gpurun_out/bcp.log
