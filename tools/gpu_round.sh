# ad-hoc GPU session script: args = test files; then the step's kernel replay
bash tools/gpu_tests.sh "$@"
timeout 600 python tools/kernel_replay.py --cublas --top 120 --json gpurun_out/replay.json > gpurun_out/replay.log 2>&1; echo replay rc=$? >> gpurun_out/replay.log
