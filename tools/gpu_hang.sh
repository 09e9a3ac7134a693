mkdir -p gpurun_out
: > gpurun_out/hang.log
for v in "X=1" "DP_TAIL_GRAPH=0" "DP_LATE_OPT_JOIN=0" "PROBE_SNAP=0" "PROBE_PREFETCH=1"; do
  echo "== $v" >> gpurun_out/hang.log
  env $v timeout -s KILL 150 python tools/hang_probe.py >> gpurun_out/hang.log 2>&1; echo "rc=$?" >> gpurun_out/hang.log
done
bash tools/gpu_fuse_ab.sh
