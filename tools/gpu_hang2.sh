# c5 full-width iteration (bench-config parity file) with / without the GELU epilogue, hard timeouts
mkdir -p gpurun_out
: > gpurun_out/hang2.log
for v in "DP_GELU_EPI=0" "X=1" "X=2"; do
  echo "== $v" >> gpurun_out/hang2.log
  env $v timeout -s KILL 420 python -m pytest tests/test_zz_bench_config_parity_gpu.py -q -x -k c5 >> gpurun_out/hang2.log 2>&1; echo "rc=$?" >> gpurun_out/hang2.log
done
timeout -s KILL 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "row_bias or geglu or bias_grad or layer_norm or ln" > gpurun_out/k2.log 2>&1; echo rc=$? >> gpurun_out/k2.log
