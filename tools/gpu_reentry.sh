# re-entry GPU check: full GPU suite, smoke, bench line, one-step ncu launch list
mkdir -p gpurun_out
bash tools/gpu_full.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/one_step.py > gpurun_out/ncu_step.log 2>&1; echo ncu rc=$? >> gpurun_out/ncu_step.log
