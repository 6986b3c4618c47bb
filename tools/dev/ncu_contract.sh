cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
A="--config c3 --c3-inst 16384 --steps 1 --warmup 1 --no-cpu"
PODECM_ROM_LAZY=1 python bench.py $A > gpurun_out/x.json 2>&1 || exit 1
for m in 0 1; do
PODECM_ROM_LAZY=$m timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rom_contract --launch-skip 20 --launch-count 1 -o gpurun_out/contract_lazy$m python bench.py $A > gpurun_out/ncu_c$m.log 2>&1
done
