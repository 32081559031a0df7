#!/bin/bash
# bf16 GEMM + layer-level check: parity subset, layer benches, stream-mix ceilings
TAG=${1:-ly}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider -x -k "gemm_bf16 or s6 or bf16" > gpurun_out/pytest_layer_$TAG.log 2>&1; tail -3 gpurun_out/pytest_layer_$TAG.log
tools/ubench/streams
for wl in s6_layer rglru_layer s6; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline --steps 5 > gpurun_out/bench_${wl}_$TAG.json 2> gpurun_out/bench_${wl}_$TAG.err
  python -c "import json; d=json.load(open('gpurun_out/bench_${wl}_$TAG.json')); print('$wl', round(d['ms_per_step'],3), round(d['value'],2), {k: round(v,3) for k,v in d['kernels'].items()}, d['roofline']['kernel'], round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2))" || tail -5 gpurun_out/bench_${wl}_$TAG.err
done
