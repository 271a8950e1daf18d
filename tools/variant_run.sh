#!/bin/bash
# usage (on the GPU box): tools/variant_run.sh [workloads...] -- time every .so in _lib/variants
W=${@:-cfg4 cfg3 cfg5}
cp paracut_b200/_lib/libparacut_b200.so /tmp/_keep.so
for v in paracut_b200/_lib/variants/*.so; do
  cp $v paracut_b200/_lib/libparacut_b200.so; echo "== $v"
  for w in $W; do timeout 120 python tools/profile_step.py --iters 20 --workload $w; done
done
cp /tmp/_keep.so paracut_b200/_lib/libparacut_b200.so
