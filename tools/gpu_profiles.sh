#!/bin/bash
# Round profile set: launch lists (all workloads) + ncu --set full of the dominant kernels.
TAG=${1:-r2a}
mkdir -p gpurun_out
for WL in ${WLS:-rglru s6 s5 lru s6_long s6_layer rglru_layer}; do
  timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/launches_${WL}_$TAG.csv python tools/prof_step.py --workload $WL --steps 2 > /dev/null 2>&1
  echo "list $WL rc=$?"
done
for spec in "s6:^(fwd|bwd)_kernel$:2" "s5:gemm:6" "rglru:(bwd_rev2|fwd2)_kernel:2" "s6_layer:gemm_bf16:1"; do
  WL=$(echo $spec | cut -d: -f1); RE=$(echo $spec | cut -d: -f2); C=$(echo $spec | cut -d: -f3)
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$RE" -s 0 -c $C \
    -o gpurun_out/prof_${WL}_$TAG python tools/prof_step.py --workload $WL --steps 1 > gpurun_out/ncu_full_${WL}_$TAG.log 2>&1
  echo "full $WL rc=$?"
done
