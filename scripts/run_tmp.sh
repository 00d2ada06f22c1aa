python -m pytest tests -m gpu -x -q > gpurun_out/gputest_merge.log 2>&1; tail -3 gpurun_out/gputest_merge.log
python bench.py --config 4 --no-cpu-baseline --no-per-config > gpurun_out/bench_c4_merge.json 2> gpurun_out/bench_c4_merge.err
python bench.py --config 3 --no-cpu-baseline --no-per-config > gpurun_out/bench_c3_merge.json 2> gpurun_out/bench_c3_merge.err
python - <<'P'
import json
for c in (4,3):
    d=json.loads([l for l in open(f'gpurun_out/bench_c{c}_merge.json') if l.startswith('{')][-1])
    print(c, d['ms_per_step'], [(x['name'], round(x['ms_per_launch']*1e3,1)) for x in d['components']])
P
mkdir -p gpurun_out/prof_merge
for k in m3_apply_kernel m4_kernel; do
ncu -f --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o /tmp/full_$k python scripts/one_solve.py 4 1 > gpurun_out/prof_merge/ncu_$k.log 2>&1
ncu -i /tmp/full_$k.ncu-rep --page raw --csv > gpurun_out/prof_merge/full_c4_$k.csv 2>/dev/null
done
