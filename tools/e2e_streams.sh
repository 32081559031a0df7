#!/bin/bash
# e2e sub-batch stream-count sweep (workload x LRX_E2E_STREAMS)
for wl in ${WLS:-rglru_layer s6_layer rglru}; do
  for ns in ${NS:-1 2 4 8 64}; do
    LRX_E2E_STREAMS=$ns timeout 900 python bench.py --workload $wl --steps 3 --no-cpu-baseline > gpurun_out/e.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/e.json')); e=d['e2e']; print('$wl streams=$ns', round(e['value'],3), round(e['ms_per_step'],1), 'ms', round((e['h2d_bytes_per_step']+e['d2h_bytes_per_step'])/e['ms_per_step']/1e6,1), 'GB/s PCIe')"
  done
done
