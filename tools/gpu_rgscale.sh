#!/bin/bash
# RG-LRU per-rank shares (B = 64/32/16/8) under plan overrides: EXTRA="cfg1|cfg2|..." (| separated)
IFS='|' read -ra CFGS <<< "${EXTRA:-}"
for cfg in "" "${CFGS[@]}"; do
  echo "== [$cfg]"; env $cfg timeout 600 python tools/scaling_probe.py rglru 2>&1 | grep "N=" | sed -n "${ROWS:-1,4}p"
done
