#!/bin/bash
# ncu: launch list + full capture of the top kernels of one workload.
WL=${1:-rglru}; TAG=${2:-r1}; REGEX=${3:-"fwd_tma|bwd_tma"}; B=${4:-0}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k "regex:kernel" --csv --log-file gpurun_out/launches_${WL}_$TAG.csv \
  python tools/prof_step.py --workload $WL --batch $B --steps 2 > gpurun_out/ncu_list_${WL}_$TAG.log 2>&1
echo "list rc=$?"; tail -2 gpurun_out/ncu_list_${WL}_$TAG.log
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$REGEX" -s 0 -c 2 \
  -o gpurun_out/prof_${WL}_$TAG python tools/prof_step.py --workload $WL --batch $B --steps 1 > gpurun_out/ncu_full_${WL}_$TAG.log 2>&1
echo "full rc=$?"; tail -3 gpurun_out/ncu_full_${WL}_$TAG.log
