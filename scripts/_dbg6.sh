for p in 2 5 10; do
  ASDSM_STRIPS=$p timeout 300 python bench.py --config 2 --no-per-config --no-cpu-baseline --steps 3 --warmup 3 > gpurun_out/bs$p.log 2>&1
  echo "strips $p rc=$?" >> gpurun_out/bc.txt
done
for p in 2 10; do
ASDSM_STRIPS=$p timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -p no:cacheprovider -k "config2" > gpurun_out/t2d$p.log 2>&1
echo "tests $p rc=$?" >> gpurun_out/bc.txt
done
