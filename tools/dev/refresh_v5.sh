cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/r1_bench_all_v5.json 2> gpurun_out/bench_v5.err; echo bench rc=$?
A="--config c3 --c3-inst 16384 --steps 1 --warmup 1 --no-cpu"
timeout 900 ncu --set full --import-source on --clock-control none -k 'regex:k_rom_(point|contract|check|solve|F)' --launch-skip 60 -c 6 -o gpurun_out/r1_c3_rom_v5 python bench.py $A > gpurun_out/ncu_c3_v5.log 2>&1; echo ncu rc=$?
