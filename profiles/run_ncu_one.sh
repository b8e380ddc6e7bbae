#!/bin/bash
# ncu --set full capture of selected kernels of one fwd+bwd step (7B shape)
# usage: run_ncu_one.sh <regex> <skip> <count> <out-name> [bench args]
K=$1; S=$2; C=$3; NAME=$4; shift 4
timeout 1500 ncu --set full --clock-control none --import-source on -k "regex:$K" -s $S -c $C \
    -o gpurun_out/$NAME -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e "$@" > gpurun_out/$NAME.log 2>&1
tail -2 gpurun_out/$NAME.log
