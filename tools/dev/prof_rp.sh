python tools/dev/c3_ab.py 8192 /tmp/x.npz > /dev/null 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_rom_contract" --launch-skip 30 --launch-count 1 -f -o gpurun_out/r2c_contract_rp python tools/dev/c3_ab.py 8192 /tmp/x.npz > gpurun_out/ncu_rp.log 2>&1
echo done
