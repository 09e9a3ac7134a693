# kernel tests for this session's changes + A/B of committed HEAD (abtest/head) vs the working tree
mkdir -p gpurun_out
timeout -s KILL 900 python -m pytest tests/test_kernels_gpu.py tests/test_gemm_gpu.py -q -x > gpurun_out/k_tests.log 2>&1; echo rc=$? >> gpurun_out/k_tests.log
timeout -s KILL 900 python -m pytest tests/test_c2_parity_gpu.py tests/test_optimizer_overlap_gpu.py tests/test_ext_configs_gpu.py -q -x > gpurun_out/p_tests.log 2>&1; echo rc=$? >> gpurun_out/p_tests.log
: > gpurun_out/ab_tree.log
for r in 1 2 3; do
  echo "== HEAD run $r" >> gpurun_out/ab_tree.log
  (cd abtest/head && timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | cut -c1-120) >> gpurun_out/ab_tree.log
  echo "== WORK run $r" >> gpurun_out/ab_tree.log
  timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | cut -c1-120 >> gpurun_out/ab_tree.log
done
timeout -s KILL 1300 python -m pytest tests/test_zz_bench_config_parity_gpu.py -q -x > gpurun_out/bcp_tests.log 2>&1; echo rc=$? >> gpurun_out/bcp_tests.log
