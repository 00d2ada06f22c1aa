for c in 0 1 2; do
  timeout 300 python bench.py --config $c --no-per-config --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/bc$c.log 2>&1
  echo "config $c rc=$?" >> gpurun_out/bc.txt
done
