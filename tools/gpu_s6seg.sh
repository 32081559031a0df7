#!/bin/bash
# S6 plan sweep on C3: time segments and forward thread width, plus the MUFU ceiling
tools/ubench/mufu2
for cfg in "LRX_S6_SEGS=1" "LRX_S6_SEGS=2" "LRX_S6_SEGS=3" "LRX_S6_SEGS=4" "LRX_S6_FWD_NPT=2" "LRX_S6_FWD_NPT=2 LRX_S6_SEGS=2"; do
  echo "== $cfg"; env $cfg timeout 300 python tools/s6_micro.py s6 2>&1 | tail -3
done
