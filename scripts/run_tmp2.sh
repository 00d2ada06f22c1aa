python -m pytest tests -m gpu -x -q -k "3d or full or hole or stages or even_odd or transform" > gpurun_out/gputest_h3.log 2>&1; tail -3 gpurun_out/gputest_h3.log
for c in 4 3 2; do python bench.py --config $c --no-cpu-baseline --no-per-config > gpurun_out/bench_c${c}_h3.json 2> gpurun_out/bench_c${c}_h3.err; done
python - <<'P'
import json
for c in (4,3,2):
    d=json.loads([l for l in open(f'gpurun_out/bench_c{c}_h3.json') if l.startswith('{')][-1])
    print(c, d['ms_per_step'], [(x['name'], round(x['ms_per_launch']*1e3,1)) for x in d['components']])
P
