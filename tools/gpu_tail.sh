mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_c2_parity_gpu.py tests/test_cuda_graph_gpu.py tests/test_c1_parity_gpu.py tests/test_zz_bench_config_parity_gpu.py -q -x > gpurun_out/tail_tests.log 2>&1; echo rc=$? >> gpurun_out/tail_tests.log
: > gpurun_out/tail_ab.log
for v in "X=1" "DP_TAIL_GRAPH=0" "X=2"; do
  echo "== $v" >> gpurun_out/tail_ab.log
  env $v timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | grep '^{' | cut -c1-100 >> gpurun_out/tail_ab.log
done
