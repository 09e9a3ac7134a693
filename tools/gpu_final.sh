# final round-2 GPU evidence: full GPU suite, smoke, bench line, one-step launch list, ncu --set full of step kernels
mkdir -p gpurun_out
bash tools/gpu_full.sh
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file gpurun_out/launches.csv python tools/one_step.py > gpurun_out/ncu_step.log 2>&1; echo ncu rc=$? >> gpurun_out/ncu_step.log
timeout 900 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:tc_gemm_kernel -s 40 -c 12 -o gpurun_out/step_gemm python tools/one_step.py > gpurun_out/ncu_gemm.log 2>&1; echo rc=$? >> gpurun_out/ncu_gemm.log
timeout 600 ncu --set full --clock-control none --import-source on --profile-from-start off -k regex:"gn_apply|gn_partial|fa_bwd_kernel|fa_fwd|bias_grad_rows|geglu_bwd_bias" -c 16 -o gpurun_out/step_misc python tools/one_step.py > gpurun_out/ncu_misc.log 2>&1; echo rc=$? >> gpurun_out/ncu_misc.log
