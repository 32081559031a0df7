#!/bin/bash
# S6 iteration: parity subset + s6 benches.  Usage: tools/gpu_s6.sh TAG
TAG=${1:-s6}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x --tb=short -p no:cacheprovider -k "${KSEL:-s6}" > gpurun_out/pytest_$TAG.log 2>&1; tail -30 gpurun_out/pytest_$TAG.log
for wl in ${WLS:-s6 s6_long}; do
  timeout 600 python bench.py --workload $wl --no-cpu-baseline --steps 5 > gpurun_out/bench_${wl}_$TAG.json 2> gpurun_out/bench_${wl}_$TAG.err
  echo "== $wl"; python -c "import json;d=json.load(open('gpurun_out/bench_${wl}_$TAG.json'));print(d['value'], d['kernels'], d['e2e']['value'])" 2>&1 | tail -2; tail -3 gpurun_out/bench_${wl}_$TAG.err
done
