python bench.py --config c3 --c3-inst 16384 --steps 1 --warmup 1 --no-cpu > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"k_rom_contract|k_rom_solve|k_rom_F|k_rom_point" -s 20 -c 8 -o gpurun_out/r2_c3 python bench.py --config c3 --c3-inst 16384 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu.log 2>&1
echo rc $?
