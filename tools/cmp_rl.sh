# compare two builds of the sweep under ncu (run on the GPU box)
mkdir -p gpurun_out
cp paracut_b200/_lib/libparacut_b200.so /tmp/base.so
for v in base rl16; do
  if [ $v = rl16 ]; then cp paracut_b200/_lib/variants/rl16.so paracut_b200/_lib/libparacut_b200.so; else cp /tmp/base.so paracut_b200/_lib/libparacut_b200.so; fi
  md5sum paracut_b200/_lib/libparacut_b200.so
  timeout 300 ncu --section SpeedOfLight --section Occupancy --section WarpStateStats --section SchedulerStats --section MemoryWorkloadAnalysis_Tables --clock-control none -k regex:k_sweep -s 7 -c 1 -o gpurun_out/cmp_$v python tools/profile_step.py --workload cfg4 > gpurun_out/cmp_$v.log 2>&1
  tail -2 gpurun_out/cmp_$v.log
done
cp /tmp/base.so paracut_b200/_lib/libparacut_b200.so
