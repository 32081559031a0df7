#!/bin/bash
# quick perf probe: rglru fwd variants + s6 bench
TAG=${1:-q}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x --tb=short -p no:cacheprovider -k "rglru or s6 or determin" > gpurun_out/pytest_$TAG.log 2>&1; tail -3 gpurun_out/pytest_$TAG.log
for m in lookback stream; do
  LRX_RGLRU_MODE=$m timeout 300 python bench.py --workload rglru --no-cpu-baseline --steps 5 > gpurun_out/bench_rglru_${m}_$TAG.json 2> gpurun_out/bench_rglru_${m}_$TAG.err
  echo "== $m"; python -c "import json;d=json.load(open('gpurun_out/bench_rglru_${m}_$TAG.json'));print(d['value'], d['kernels'], d['e2e']['value'])" 2>&1 | tail -2
done
timeout 300 python bench.py --workload s6 --no-cpu-baseline --steps 5 > gpurun_out/bench_s6_$TAG.json 2> gpurun_out/bench_s6_$TAG.err
echo "== s6"; python -c "import json;d=json.load(open('gpurun_out/bench_s6_$TAG.json'));print(d['value'], d['kernels'])" 2>&1 | tail -2; tail -2 gpurun_out/bench_s6_$TAG.err
