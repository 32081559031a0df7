#!/bin/bash
# MIMO (S5 / LRU) step under GEMM plan overrides: bench ms/step per setting
for wl in ${WLS:-lru s5}; do
  for cfg in "" "LRX_GEMM_BN=64" "LRX_GEMM_TN_CTAS=16" "LRX_GEMM_TN_CTAS=32" "LRX_GEMM_TN_CTAS=64" ${EXTRA}; do
    env $cfg timeout 600 python bench.py --workload $wl --steps 20 --no-cpu-baseline > gpurun_out/m.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/m.json')); print('$wl', '${cfg:-default}', round(d['ms_per_step']*1e3,1), 'us/step', round(d['value'],1), d['unit'])"
  done
done
