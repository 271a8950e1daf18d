#!/bin/bash
# usage (on the GPU box): tools/variant_run.sh [workloads...] -- steady-state time of every .so in _lib/variants
W=${@:-cfg4 cfg3 cfg5}
cp paracut_b200/_lib/libparacut_b200.so /tmp/_keep.so
for rep in 1 2; do
for v in paracut_b200/_lib/variants/*.so; do
  cp $v paracut_b200/_lib/libparacut_b200.so; echo "== $v"
  for w in $W; do timeout 300 python tools/ab_steady.py $w; done
done
done
cp /tmp/_keep.so paracut_b200/_lib/libparacut_b200.so
