#!/bin/bash
# S5 / LRU step: separate launches vs fused forward vs fused forward + backward
for wl in ${WLS:-s5}; do
  for cfg in "LRX_MIMO_FUSED=0" "LRX_MIMO_FUSED=1" "LRX_MIMO_FUSED=1 LRX_MIMO_FUSED_BWD=1"; do
    env $cfg timeout 600 python bench.py --workload $wl --steps ${STEPS:-20} --no-cpu-baseline > /tmp/ab.json 2>/dev/null
    python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$wl', '$cfg', round(d['ms_per_step']*1e3,1), 'us/step fwd', round(k['fwd_ms']*1e3,1), 'bwd', round(k['bwd_ms']*1e3,1))"
  done
done
