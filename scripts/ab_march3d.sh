for v in "" "ASDSM_MARCH3D=1"; do for c in 3 4; do env $v python bench.py --config $c --no-cpu-baseline --steps 3 --no-all-configs 2>&1 | tail -1 > gpurun_out/b.json; echo "== $v config $c"; python -c "
import json; d=json.load(open('gpurun_out/b.json'))
print('ms %.3f'%(d['ms_per_step']))
[print('%-26s %8.1f us %s'%(c['name'],c['ms_per_launch']*1e3, c['gbs'])) for c in d['components'] if c['name'] in ('update_residual','step_dots','residual')]
"; done; done
