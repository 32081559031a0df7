#!/bin/bash
# fused projection + scan (default) vs separate GEMM + scan launches (LRX_MIMO_FUSED=0)
for wl in ${WLS:-s5 lru}; do
  for i in 1 2; do
    for f in 1 0; do
      LRX_MIMO_FUSED=$f timeout 600 python bench.py --workload $wl --steps ${STEPS:-20} --no-cpu-baseline > /tmp/ab.json 2>/dev/null
      python -c "import json; d=json.load(open('/tmp/ab.json')); k=d['kernels']; print('$wl fused=$f', round(d['ms_per_step']*1e3,1), 'us/step fwd', round(k['fwd_ms']*1e3,1), 'bwd', round(k['bwd_ms']*1e3,1), 'launches', d['gpu_launches'])"
    done
  done
done
