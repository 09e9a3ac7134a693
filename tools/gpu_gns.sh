mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x -k "groupnorm_statistics or conv_implicit" > gpurun_out/gns_tests.log 2>&1; echo rc=$? >> gpurun_out/gns_tests.log
timeout 600 python -m pytest tests/test_c2_parity_gpu.py tests/test_zz_bench_config_parity_gpu.py -q -x > gpurun_out/gns_parity.log 2>&1; echo rc=$? >> gpurun_out/gns_parity.log
: > gpurun_out/gns_ab.log
for v in "X=1" "DP_GN_STATS=0" "X=2" "DP_GN_STATS=0"; do
  echo "== $v" >> gpurun_out/gns_ab.log
  env $v timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | cut -c1-100 >> gpurun_out/gns_ab.log
done
