# the driver's GPU test tier as it runs it: ONE pytest process over every -m gpu test, then smoke
mkdir -p gpurun_out
timeout -s KILL 2700 python -m pytest tests/ -x -q -m gpu > gpurun_out/driver_tests.log 2>&1; echo rc=$? >> gpurun_out/driver_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke.log
