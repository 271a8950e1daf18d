#!/bin/bash
# usage (GPU box): tools/vp_variants.sh WL ITERS WIN -- verify_phase for the main .so and every variant
cp paracut_b200/_lib/libparacut_b200.so /tmp/_keep.so
echo "== main"; python tools/verify_phase.py "$@"
for v in paracut_b200/_lib/variants/*.so; do
  cp $v paracut_b200/_lib/libparacut_b200.so; echo "== $v"; python tools/verify_phase.py "$@"
done
cp /tmp/_keep.so paracut_b200/_lib/libparacut_b200.so
