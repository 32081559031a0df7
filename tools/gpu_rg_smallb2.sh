#!/bin/bash
BS="32" ; for cfg in "LRX_RGLRU_PF=4" "LRX_RGLRU_PF=8" "LRX_RGLRU_PF=4 LRX_RGLRU_STAGES=4" "LRX_RGLRU_PF=4 LRX_RGLRU_STAGES=3" "LRX_RGLRU_PF=8 LRX_RGLRU_STAGES=3"; do
  env $cfg timeout 300 python tools/rg_smallb.py $BS 2>&1 | grep "^B="; done
BS="16" ; for cfg in "LRX_RGLRU_PF=8" "LRX_RGLRU_PF=16" "LRX_RGLRU_PF=8 LRX_RGLRU_STAGES=3" "LRX_RGLRU_PF=8 LRX_RGLRU_STAGES=8"; do
  env $cfg timeout 300 python tools/rg_smallb.py $BS 2>&1 | grep "^B="; done
BS="8" ; for cfg in "LRX_RGLRU_SEGS=1" "LRX_RGLRU_SEGS=3 LRX_RGLRU_PF=4" "LRX_RGLRU_SEGS=3 LRX_RGLRU_PF=16" "LRX_RGLRU_SEGS=2 LRX_RGLRU_PF=16" "LRX_RGLRU_SEGS=1 LRX_RGLRU_PF=16"; do
  env $cfg timeout 300 python tools/rg_smallb.py $BS 2>&1 | grep "^B="; done
BS="64" ; for cfg in "" "LRX_RGLRU_PF=4"; do
  env $cfg timeout 300 python tools/rg_smallb.py $BS 2>&1 | grep "^B="; done
