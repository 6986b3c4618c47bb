cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python bench.py > gpurun_out/r1_bench_all_v9.json 2> gpurun_out/bench_v9.err; echo bench rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r1_launches_c1_v9.csv python bench.py --config c1 --steps 2 --warmup 3 --no-cpu > gpurun_out/ncu_launch_v9.log 2>&1; echo launch rc=$?
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_material --launch-skip 3 --launch-count 1 -o gpurun_out/r1_c1_material_v9 python bench.py --config c1 --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_c1_v9.log 2>&1; echo ncu1 rc=$?
