# the round-end driver's GPU tiers as it runs them: ONE pytest process over every -m gpu test, smoke, bench
mkdir -p gpurun_out
timeout -s KILL 2700 python -m pytest tests/ -x -q -m gpu > gpurun_out/driver_tests.log 2>&1; echo rc=$? >> gpurun_out/driver_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$? >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo bench rc=$? >> gpurun_out/bench.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/one_step.py > gpurun_out/ncu_step.log 2>&1; echo ncu rc=$? >> gpurun_out/ncu_step.log
python tools/ncu_summary.py launches gpurun_out/launches.csv > gpurun_out/launches.txt 2>&1 && rm -f gpurun_out/launches.csv
timeout 900 ncu --set full --clock-control none --profile-from-start off -k regex:tc_gemm_kernel -s 40 -c 8 -o /tmp/step_gemm python tools/one_step.py > gpurun_out/ncu_gemm.log 2>&1; echo rc=$? >> gpurun_out/ncu_gemm.log
python tools/ncu_summary.py full /tmp/step_gemm.ncu-rep > gpurun_out/ncu_full_gemm.txt 2>&1
timeout 600 ncu --set full --clock-control none --profile-from-start off -k regex:"gn_apply|gn_partial|fa_bwd_kernel|fa_fwd|geglu_bwd_bias" -c 10 -o /tmp/step_misc python tools/one_step.py > gpurun_out/ncu_misc.log 2>&1; echo rc=$? >> gpurun_out/ncu_misc.log
python tools/ncu_summary.py full /tmp/step_misc.ncu-rep > gpurun_out/ncu_full_misc.txt 2>&1
