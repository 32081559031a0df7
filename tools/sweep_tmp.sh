tools/ncu_one.sh rglru bwd_rev r2rev 1
for cfg in "" "LRX_RGLRU_PF=8" "LRX_RGLRU_STAGES=3" "LRX_RGLRU_LW=64" "LRX_RGLRU_LW=64 LRX_RGLRU_STAGES=3" "LRX_RGLRU_PF=8 LRX_RGLRU_LW=64"; do
  env $cfg timeout 300 python bench.py --workload rglru --no-cpu-baseline > gpurun_out/sw.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('$cfg', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernels'].items()}, round(d['roofline']['per_launch_ms'],3))"
done
