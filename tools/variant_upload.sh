cp paracut_b200/_lib/libparacut_b200.so /tmp/_keep.so
for v in paracut_b200/_lib/variants/*.so; do
  cp $v paracut_b200/_lib/libparacut_b200.so; echo "== $v"
  timeout 300 python tools/upload_probe.py cfg5
done
cp /tmp/_keep.so paracut_b200/_lib/libparacut_b200.so
