#!/bin/bash
# usage (GPU box): tools/bench_all.sh OUTDIR -- bench lines of every BASELINE workload / mode
cd $GRAFT_REPO_ROOT
O=${1:-gpurun_out/all}; mkdir -p $O
run() { n=$1; shift; timeout 900 python bench.py "$@" > $O/$n.json 2> $O/$n.err; }
run cfg4 --steps 20 --warmup 5
run cfg1_f64 --workload cfg1 --precision f64 --steps 20 --warmup 5 --no-ttc
run cfg1_f64s --workload cfg1 --precision f64s --steps 20 --warmup 5 --no-ttc
run cfg2 --workload cfg2 --steps 20 --warmup 5
run cfg3 --workload cfg3 --steps 20 --warmup 5 --no-ttc
run cfg4_f64s --precision f64s --steps 20 --warmup 5 --no-ttc --no-cpu
run cfg4_f64 --precision f64 --steps 20 --warmup 5 --no-ttc --no-cpu
run cfg5 --workload cfg5 --steps 10 --warmup 5 --no-ttc --cpu-iters 1
run cfg4_sharded --sharded --steps 20 --warmup 5
run ref_cfg4 --impl reference --steps 5 --warmup 1
timeout 600 python tools/virtual_shard_bench.py cfg4 > $O/virtual_cfg4.txt 2>&1
