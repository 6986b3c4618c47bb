python bench.py --config c2 --c2-inst 128 --steps 1 --warmup 1 --no-cpu > gpurun_out/plain_c2.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_asm_qp2" --launch-skip 2 --launch-count 1 -o gpurun_out/r2b_c2 python bench.py --config c2 --c2-inst 128 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_c2.log 2>&1
echo done
