cp paracut_b200/_lib/libparacut_b200.so /tmp/_keep.so
for v in paracut_b200/_lib/variants/*.so; do
  cp $v paracut_b200/_lib/libparacut_b200.so; echo "== $v"
  for w in cfg1 cfg2 cfg4; do timeout 120 python tools/profile_step.py --iters 10 --workload $w --precision f64; done
done
cp /tmp/_keep.so paracut_b200/_lib/libparacut_b200.so
