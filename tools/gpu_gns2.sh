mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_zz_bench_config_parity_gpu.py -v -x > gpurun_out/gns_parity.log 2>&1; echo rc=$? >> gpurun_out/gns_parity.log
DP_GN_STATS=1 timeout 600 python -m pytest tests/test_c2_parity_gpu.py tests/test_zz_bench_config_parity_gpu.py -v -x -k "c2" > gpurun_out/gns_parity_on.log 2>&1; echo rc=$? >> gpurun_out/gns_parity_on.log
