mkdir -p gpurun_out
timeout -s KILL 2000 python -m pytest tests/ -x -q -m gpu > gpurun_out/driver_tests2.log 2>&1; echo rc=$? >> gpurun_out/driver_tests2.log
timeout 900 python bench.py > gpurun_out/bench2.log 2>&1; echo bench rc=$? >> gpurun_out/bench2.log
