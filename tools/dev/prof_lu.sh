python tools/dev/c3_ab.py 4096 /tmp/x.npz > gpurun_out/plain_lu.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_rom_solve" --launch-skip 20 --launch-count 1 -o gpurun_out/r2_lu_reg python tools/dev/c3_ab.py 4096 /tmp/x.npz > gpurun_out/ncu_lu.log 2>&1
PODECM_ROM_LU=smem ncu --set full --clock-control none --import-source on -k regex:"k_rom_solve" --launch-skip 20 --launch-count 1 -o gpurun_out/r2_lu_smem python tools/dev/c3_ab.py 4096 /tmp/x.npz > gpurun_out/ncu_lu2.log 2>&1
echo done
