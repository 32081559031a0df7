#!/bin/bash
# One gpurun session: parity suite, smoke, every bench line.  Usage: tools/gpu_session.sh TAG [workloads...]
TAG=${1:-r2}; shift
WLS=${@:-rglru s6 s5 lru s6_long s6_layer rglru_layer}
mkdir -p gpurun_out/bench_$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/bench_$TAG/gpu.txt
if [ -z "$NO_TESTS" ]; then
  timeout 1500 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/bench_$TAG/pytest_gpu.log 2>&1
  tail -3 gpurun_out/bench_$TAG/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/bench_$TAG/smoke.log 2>&1; tail -2 gpurun_out/bench_$TAG/smoke.log
fi
for wl in $WLS; do
  timeout 900 python bench.py --workload $wl > gpurun_out/bench_$TAG/bench_${wl}.json 2> gpurun_out/bench_$TAG/bench_${wl}.err
  echo "== $wl rc=$?"; python -c "import json; d=json.load(open('gpurun_out/bench_$TAG/bench_${wl}.json')); print(round(d['value'],2), d['unit'], round(d['ms_per_step'],3), 'ms', d['roofline']['kernel'][:40], 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value'],2), 'cpu', d['cpu_baseline'] and round(d['cpu_baseline']['value'],4))" 2>&1 | tail -1
  timeout 900 python bench.py --workload $wl --impl reference --steps 2 --warmup 1 > gpurun_out/bench_$TAG/ref_${wl}.json 2> gpurun_out/bench_$TAG/ref_${wl}.err
done
