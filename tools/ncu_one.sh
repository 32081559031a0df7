#!/bin/bash
# One ncu --set full capture of a kernel of a bench workload's step.
# Usage: tools/ncu_one.sh WORKLOAD KERNEL_REGEX TAG [COUNT] [extra env assignments...]
WL=$1; RE=$2; TAG=$3; C=${4:-1}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$RE" -s 0 -c $C \
  -o gpurun_out/prof_${WL}_$TAG python tools/prof_step.py --workload $WL --steps 1 > gpurun_out/ncu_${WL}_$TAG.log 2>&1
echo "ncu $WL $TAG rc=$?"
