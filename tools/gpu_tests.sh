#!/bin/bash
# Run GPU test files one by one with hard timeouts; summary to gpurun_out/tests.log
mkdir -p gpurun_out
: > gpurun_out/tests.log
for f in "$@"; do
  timeout -s KILL 1500 python -m pytest "$f" -v -x --timeout 1200 --timeout-method thread > gpurun_out/$(basename $f .py).log 2>&1
  echo "== $f rc=$?" >> gpurun_out/tests.log
  grep -E "PASSED|FAILED|ERROR|Timeout|Error|error|assert" gpurun_out/$(basename $f .py).log | head -40 >> gpurun_out/tests.log
done
cat gpurun_out/tests.log
