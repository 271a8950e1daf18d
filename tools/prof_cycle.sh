#!/bin/bash
# usage: tools/prof_cycle.sh NAME [profile_step args]  -- run on the GPU box via gpurun
NAME=$1; shift
python tools/profile_step.py "$@" > gpurun_out/${NAME}_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KERNEL:-k_sweep} -s ${SKIP:-6} -c 1 -o gpurun_out/${NAME} python tools/profile_step.py "$@" > gpurun_out/${NAME}_ncu.log 2>&1
tail -1 gpurun_out/${NAME}_ncu.log
