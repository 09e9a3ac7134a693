mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gemm_gpu.py -q -x -k conv > gpurun_out/wg_tests.log 2>&1; echo rc=$? >> gpurun_out/wg_tests.log
: > gpurun_out/wg_ab.log
for v in "X=1" "DP_WGRAD_BN128=1"; do
  echo "== $v" >> gpurun_out/wg_ab.log
  env $v timeout 600 python tools/conv_bench.py --no-cudnn 2>&1 | cut -c1-220 >> gpurun_out/wg_ab.log
done
