#!/bin/bash
# Round profile set: launch lists + ncu --set full of the top kernels per workload.
TAG=${1:-r1e}
mkdir -p gpurun_out
for spec in "s6:^(fwd|bwd)_kernel$" "s6_long:^(fwd|bwd)(_agg)?_kernel$" "rglru:fwd_tma|bwd_tma" "s5:mimo|reduce_rows|sgemm" ; do
  WL=${spec%%:*}; RE=${spec#*:}
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_${WL}_$TAG.csv python tools/prof_step.py --workload $WL --steps 2 > /dev/null 2>&1
  echo "list $WL rc=$?"
done
for spec in "s6:^(fwd|bwd)_kernel$:2" "s6_long:^(fwd|bwd)_agg_kernel$:2" ; do
  WL=$(echo $spec | cut -d: -f1); RE=$(echo $spec | cut -d: -f2); C=$(echo $spec | cut -d: -f3)
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$RE" -s 0 -c $C \
    -o gpurun_out/prof_${WL}_$TAG python tools/prof_step.py --workload $WL --steps 1 > gpurun_out/ncu_full_${WL}_$TAG.log 2>&1
  echo "full $WL rc=$?"
done
