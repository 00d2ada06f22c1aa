export ASDSM_S3_PROBE=2
python scripts/one_solve.py 4 1 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:stream3d -s 2 -c 1 -o gpurun_out/s3prof4 python scripts/one_solve.py 4 1 > gpurun_out/ncu.log 2>&1
