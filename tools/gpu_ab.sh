#!/bin/bash
# A/B of the working tree against a baseline copy in _ab/base (same box, alternating runs)
for wl in ${WLS:-lru s5}; do
  for i in 1 2 3; do
    for arm in base new; do
      if [ $arm = base ]; then dir=_ab/base; else dir=.; fi
      (cd $dir && env $CFG timeout 600 python bench.py --workload $wl --steps ${STEPS:-20} --no-cpu-baseline > /tmp/ab.json 2>/dev/null)
      python -c "import json; d=json.load(open('/tmp/ab.json')); print('$wl', '$arm', round(d['ms_per_step']*1e3,1), 'us/step fwd', round(d['kernels']['fwd_ms']*1e3,1), d.get('roofline',{}).get('per_launch_ms'))"
    done
  done
done
