#!/bin/bash
# RG-LRU per-rank shares (B = 64/32/16/8) under plan overrides
for cfg in "" ${EXTRA}; do
  echo "== [$cfg]"; env $cfg timeout 600 python tools/scaling_probe.py rglru 2>&1 | grep "N="
done
