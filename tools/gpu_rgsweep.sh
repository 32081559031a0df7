#!/bin/bash
# RG-LRU C4 plan sweep (env overrides), kernel times from the bench line
for cfg in "" "LRX_RGLRU_FWD_PF=2 LRX_RGLRU_FWD_STAGES=2" "LRX_RGLRU_FWD_PF=2 LRX_RGLRU_FWD_STAGES=3" "LRX_RGLRU_FWD_PF=4 LRX_RGLRU_FWD_STAGES=2" "LRX_RGLRU_FWD_PF=2 LRX_RGLRU_FWD_STAGES=4" "LRX_RGLRU_BWD_PF=2 LRX_RGLRU_BWD_STAGES=2" "LRX_RGLRU_BWD_PF=2 LRX_RGLRU_BWD_STAGES=3" "LRX_RGLRU_BWD_PF=2 LRX_RGLRU_BWD_STAGES=4" ${EXTRA}; do
  env $cfg timeout 300 python bench.py --workload rglru --no-cpu-baseline --steps 5 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('[$cfg]', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernels'].items()}, 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/sw.err
done
