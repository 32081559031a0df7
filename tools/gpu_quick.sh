#!/bin/bash
# quick perf probe: parity subset + rglru variants + s6 bench
TAG=${1:-q}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider -k "${KSEL:-rglru or s6 or determin or native}" > gpurun_out/pytest_$TAG.log 2>&1; tail -15 gpurun_out/pytest_$TAG.log
for m in ${MODES:-auto stream}; do
  LRX_RGLRU_MODE=$m timeout 300 python bench.py --workload rglru --no-cpu-baseline --steps 5 > gpurun_out/bench_rglru_${m}_$TAG.json 2> gpurun_out/bench_rglru_${m}_$TAG.err
  echo "== $m"; python -c "import json;d=json.load(open('gpurun_out/bench_rglru_${m}_$TAG.json'));print(d['value'], d['kernels'], d['e2e']['value'])" 2>&1 | tail -2; tail -2 gpurun_out/bench_rglru_${m}_$TAG.err
done
for wl in ${WLS:-s6}; do
timeout 300 python bench.py --workload $wl --no-cpu-baseline --steps 5 > gpurun_out/bench_${wl}_$TAG.json 2> gpurun_out/bench_${wl}_$TAG.err
echo "== $wl"; python -c "import json;d=json.load(open('gpurun_out/bench_${wl}_$TAG.json'));print(d['value'], d['kernels'])" 2>&1 | tail -2; tail -2 gpurun_out/bench_${wl}_$TAG.err
done
