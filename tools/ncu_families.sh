#!/bin/bash
# On the GPU box: ncu --set full of one iteration's family sweeps of a workload
# (after 2 warm-up iterations); details + raw CSV under gpurun_out/fam_<wl>/.
WL=$1; NF=$2
O=gpurun_out/fam_$WL; mkdir -p $O
timeout 1200 ncu --set full --clock-control none -k regex:k_sweep -s $((2 * NF)) -c $NF \
  -o $O/rep python tools/profile_step.py --workload $WL --iters 3 > $O/ncu.log 2>&1
ncu -i $O/rep.ncu-rep --page details --csv > $O/details.csv 2>/dev/null
ncu -i $O/rep.ncu-rep --page raw --csv > $O/raw.csv 2>/dev/null
rm -f $O/rep.ncu-rep
