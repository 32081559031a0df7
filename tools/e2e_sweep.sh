for cfg in "--e2e-batch 8" "--e2e-batch 16" "--e2e-batch 64 LRX_E2E_ROWS=1" "--e2e-batch 64 LRX_E2E_ROWS=2" "--e2e-batch 32"; do
  set -- $cfg
  if [ -n "$3" ]; then export $3; else unset LRX_E2E_ROWS; fi
  timeout 600 python bench.py $1 $2 --steps 3 --no-cpu-baseline > gpurun_out/e.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/e.json')); e=d['e2e']; print('$cfg', round(e['value'],2), round(e['ms_per_step'],1), e['sample'][:40], round((e['h2d_bytes_per_step']+e['d2h_bytes_per_step'])/e['ms_per_step']/1e6,1), 'GB/s total')"
done
