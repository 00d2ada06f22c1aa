export ASDSM_STRIPS=5
python scripts/one_solve.py 2 1 > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2_strips.csv python scripts/one_solve.py 2 1 > gpurun_out/ncu.log 2>&1
