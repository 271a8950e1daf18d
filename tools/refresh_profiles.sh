#!/bin/bash
# On the GPU box: bench lines for every config, the reference arm, the cfg4
# launch list and one ncu --set full capture of the three cfg4 family sweeps.
# Outputs under gpurun_out/refresh/ (copied into profiles/ by hand).
O=gpurun_out/refresh; mkdir -p $O
timeout 600 python bench.py > $O/bench_cfg4.json 2> $O/bench_cfg4.err
for w in cfg3 cfg5 cfg2 cfg1; do
  timeout 600 python bench.py --workload $w --no-ttc > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 600 python bench.py --precision f64 --no-ttc > $O/bench_cfg4_f64.json 2> $O/bench_cfg4_f64.err
timeout 600 python bench.py --impl reference > $O/bench_reference_cfg4.json 2> $O/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches_cfg4.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-ttc > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_sweep -s 6 -c 3 \
  -o $O/full_cfg4 python tools/profile_step.py --workload cfg4 --iters 3 > $O/ncu_full.log 2>&1
ncu -i $O/full_cfg4.ncu-rep --page details --csv > $O/full_cfg4_details.csv 2>/dev/null
ncu -i $O/full_cfg4.ncu-rep --page raw --csv > $O/full_cfg4_raw.csv 2>/dev/null
rm -f $O/full_cfg4.ncu-rep
tail -n 2 $O/*.err | head -40
