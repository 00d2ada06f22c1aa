python -m pytest tests -m gpu -x -q -k "not 3d" > gpurun_out/gputest_2d.log 2>&1; tail -3 gpurun_out/gputest_2d.log
for c in 2 1; do python bench.py --config $c --no-cpu-baseline --no-per-config > gpurun_out/bench_c${c}_h3.json 2> gpurun_out/bench_c${c}_h3.err; done
python - <<'P'
import json
for c in (2,1):
    d=json.loads([l for l in open(f'gpurun_out/bench_c{c}_h3.json') if l.startswith('{')][-1])
    print(c, d['ms_per_step'], [(x['name'], round(x['ms_per_launch']*1e3,1)) for x in d['components']])
P
