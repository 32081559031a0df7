#!/bin/bash
# RG-LRU per-rank-share plan sweep (B = 32, 16, 8)
for cfg in "" "LRX_RGLRU_SCALAR=1" "LRX_RGLRU_STAGES=2" "LRX_RGLRU_STAGES=4" "LRX_RGLRU_PF=4" "LRX_RGLRU_SEGS=2" "LRX_RGLRU_SEGS=4" "LRX_RGLRU_SCALAR=1 LRX_RGLRU_SEGS=2" ${EXTRA}; do
  env $cfg timeout 300 python tools/rg_smallb.py ${BS:-32 16 8} 2>&1 | grep "^B="
done
