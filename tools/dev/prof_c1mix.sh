python bench.py --config c1 --steps 3 --warmup 3 --no-cpu > /dev/null 2>&1 || exit 1
ncu --section InstructionStats --clock-control none -k regex:k_material --launch-skip 3 --launch-count 1 -o gpurun_out/r2b_c1_mix python bench.py --config c1 --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_c1mix.log 2>&1
echo done
