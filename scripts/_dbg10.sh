ASDSM_STREAM3D=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -x -q -p no:cacheprovider -k "3d or config3 or config4 or cfg:3 or cfg:4 or ex:4" > gpurun_out/t3d_all.log 2>&1
echo "tests3d rc=$?" >> gpurun_out/ab.txt
bash scripts/_ab.sh ASDSM_STREAM3D=1 4 3
