# A/B of an env switch on bench configs: scripts/ab_switch.sh "VAR=val" configs...
sw="$1"; shift
for c in "$@"; do
  for v in base sw base sw; do
    if [ $v = sw ]; then env $sw timeout 300 python bench.py --config $c --no-per-config --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/ab_${c}_$v.log 2>&1
    else timeout 300 python bench.py --config $c --no-per-config --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/ab_${c}_$v.log 2>&1; fi
    python -c "import json;d=json.loads(open('gpurun_out/ab_${c}_$v.log').read().strip().split('\n')[-1]);print('$c $v', round(d['ms_per_step'],4))" >> gpurun_out/ab.txt
  done
done
