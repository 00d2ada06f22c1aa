#!/bin/bash
# A/B of env variants on one config: ./scripts/ab_env.sh CONFIG "VAR=a" "VAR=b" ...
c=$1; shift
for v in "$@"; do
  env $v timeout 300 python bench.py --config $c --no-all-configs --no-cpu-baseline --steps 3 > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/ab.json'))
print('config $c $v: solve %.3f ms  ' % d['ms_per_step'] + '  '.join('%s %.1f' % (x['name'], x['ms_per_launch']*1e3) for x in d['components']))"
done
