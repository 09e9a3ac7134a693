# A/B of two libdpipe builds on one box: abtest/lib_a.so vs abtest/lib_b.so, attention micro-benchmark x2 each
mkdir -p gpurun_out
: > gpurun_out/ab.log
for r in 1 2; do for v in a b; do
  echo "== $v run $r" >> gpurun_out/ab.log
  DP_LIB_PATH=abtest/lib_$v.so timeout 300 python tools/attn_bench.py 2>&1 | cut -c1-160 >> gpurun_out/ab.log
done; done
