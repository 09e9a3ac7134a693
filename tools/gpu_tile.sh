mkdir -p gpurun_out
: > gpurun_out/tile_ab.log
for v in "X=1" "DP_TILE_FEED=64" "DP_TILE_FEED=56"; do
  echo "== $v" >> gpurun_out/tile_ab.log
  env $v timeout 600 python tools/gemm_bench.py --only fwd,dgrad 2>&1 | cut -c1-200 >> gpurun_out/tile_ab.log
done
