mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo rc=$? >> gpurun_out/bench.log
for c in c3 c4 c5; do timeout 900 python bench.py --config $c --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/bench_$c.log 2>&1; done
