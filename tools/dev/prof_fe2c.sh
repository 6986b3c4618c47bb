ncu --set full --clock-control none --import-source on -k regex:"k_rom_contract" --launch-skip 200 --launch-count 1 -o gpurun_out/r2c_fe2_rp python bench.py --config fe2 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_fe2a.log 2>&1
PODECM_ROM_CONTRACT=std ncu --set full --clock-control none --import-source on -k regex:"k_rom_contract" --launch-skip 200 --launch-count 1 -o gpurun_out/r2c_fe2_std python bench.py --config fe2 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_fe2b.log 2>&1
echo done
