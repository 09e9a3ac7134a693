mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/wg_tests.log 2>&1; echo rc=$? >> gpurun_out/wg_tests.log
: > gpurun_out/wg_ab2.log
for v in "X=1" "DP_WG_NARROW=1"; do
  echo "== $v" >> gpurun_out/wg_ab2.log
  env $v timeout 600 python tools/gemm_bench.py --only wgrad 2>&1 | cut -c1-200 >> gpurun_out/wg_ab2.log
done
