#!/bin/bash
# compute-sanitizer over every kernel family (tools/sanitize_run.py), one
# log per tool under gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = memcheck ] && extra="--leak-check no"
  timeout 1500 $CS --tool $tool $extra --print-limit 50 python tools/sanitize_run.py "$@" > gpurun_out/sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/sanitize_$tool.log
done
