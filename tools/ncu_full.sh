#!/bin/bash
# ncu --set full of the round's top kernels (one GPU, single process).
# The .ncu-rep stays on the box (/tmp); its raw/details/source pages come back as CSV.
# usage: tools/ncu_full.sh <tag> <kernel-regex> <count> <bench args...>
TAG=${1:-full}; KRE=${2:-"k_pacm64|k_pacm_tc|k_draft_cost|k_sel_finalize"}; CNT=${3:-8}; shift 3
mkdir -p gpurun_out
REP=/tmp/$TAG
timeout 1200 ncu --set full --import-source on --clock-control none $NCU_EXTRA -k regex:"$KRE" -c $CNT \
  -o $REP -f python bench.py --steps 1 --warmup 3 --no-cpu "$@" > gpurun_out/ncu_$TAG.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_$TAG.log
ncu -i $REP.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>>gpurun_out/ncu_$TAG.log
ncu -i $REP.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>>gpurun_out/ncu_$TAG.log
ncu -i $REP.ncu-rep --page source --csv --print-source sass > gpurun_out/${TAG}_source.csv 2>>gpurun_out/ncu_$TAG.log
ls -la gpurun_out >> gpurun_out/ncu_$TAG.log
