mkdir -p gpurun_out
timeout 600 python tools/host_overhead.py > gpurun_out/host_overhead.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/one_step.py > gpurun_out/ncu_step.log 2>&1
