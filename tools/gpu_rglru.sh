#!/bin/bash
# RG-LRU check: parity subset, then the C4 bench with the lane-pair kernels vs the scalar ones
TAG=${1:-rg}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider -x -k "rglru" > gpurun_out/pytest_rglru_$TAG.log 2>&1; tail -3 gpurun_out/pytest_rglru_$TAG.log
for cfg in "" "LRX_RGLRU_SCALAR=1" ${EXTRA_CFGS}; do
  env $cfg timeout 300 python bench.py --workload ${WL:-rglru} --no-cpu-baseline --steps 10 > gpurun_out/sw.json 2>gpurun_out/sw.err
  python -c "import json; d=json.load(open('gpurun_out/sw.json')); print('[$cfg]', round(d['ms_per_step'],3), {k: round(v,3) for k,v in d['kernels'].items()}, 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" || tail -3 gpurun_out/sw.err
done
