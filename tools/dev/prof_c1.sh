set -e
python -m pytest tests/test_gpu_gmath.py tests/test_gpu_material_fullscale.py -q -p no:cacheprovider 2>&1 | tail -2
python bench.py --config c1 --steps 20 --warmup 3 --no-cpu > gpurun_out/r2_c1_plain.json 2>gpurun_out/r2_c1_plain.err
tail -c 700 gpurun_out/r2_c1_plain.json | head -c 700; echo
python bench.py --config c1 --steps 3 --warmup 3 --no-cpu > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_material --launch-skip 3 --launch-count 1 -o gpurun_out/r2_c1_material python bench.py --config c1 --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu.log 2>&1
echo ncu rc $?
