# kernel replay (per-signature device times vs cuBLAS) + one-step ncu launch list
mkdir -p gpurun_out
timeout 900 python tools/kernel_replay.py --cublas --top 200 --json gpurun_out/replay.json > gpurun_out/replay.log 2>&1; echo replay rc=$? >> gpurun_out/replay.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/one_step.py > gpurun_out/ncu_step.log 2>&1; echo ncu rc=$? >> gpurun_out/ncu_step.log
