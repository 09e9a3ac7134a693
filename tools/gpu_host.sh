mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gemm_gpu.py -q -x > gpurun_out/q_tests.log 2>&1; echo rc=$? >> gpurun_out/q_tests.log
echo "== HEAD" > gpurun_out/host_ab.log
(cd abtest/head && timeout 300 python tools/host_overhead.py) >> gpurun_out/host_ab.log 2>&1
echo "== WORK" >> gpurun_out/host_ab.log
timeout 300 python tools/host_overhead.py >> gpurun_out/host_ab.log 2>&1
bash tools/gpu_ab_tree.sh
