for v in "" "ASDSM_SMALL_SMEM=1"; do env $v python bench.py --config 1 --no-cpu-baseline --steps 3 2>&1 | tail -1 > gpurun_out/b.json; echo "== $v"; python -c "
import json; d=json.load(open('gpurun_out/b.json'))
print('c1 ms %.3f'%(d['ms_per_step']))
[print('%-26s %8.1f us'%(c['name'],c['ms_per_launch']*1e3)) for c in d['components']]
"; done
