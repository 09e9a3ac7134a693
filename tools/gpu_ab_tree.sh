# A/B of two source trees on one box: abtest/head (committed HEAD) vs the working tree
mkdir -p gpurun_out
: > gpurun_out/ab_tree.log
for r in 1 2; do
  echo "== HEAD run $r" >> gpurun_out/ab_tree.log
  (cd abtest/head && timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | cut -c1-120) >> gpurun_out/ab_tree.log
  echo "== WORK run $r" >> gpurun_out/ab_tree.log
  timeout 400 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep '^{' | cut -c1-120 >> gpurun_out/ab_tree.log
done
