# round-2 (session 2) evidence refresh: tests, full bench, reference arm, ncu of the new kernels
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2b_gputest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/r2b_gputest.log
python __graft_entry__.py --smoke > gpurun_out/r2b_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/r2b_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2b_bench_all.json 2> gpurun_out/r2b_bench_all.err; echo "bench rc $?"
python -c "import json; d=json.loads(open('gpurun_out/r2b_bench_all.json').read().strip().splitlines()[-1]); print(json.dumps(d['baseline_metrics']))"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2b_bench_ref.json 2>&1; echo "ref rc $?"; tail -c 600 gpurun_out/r2b_bench_ref.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2b_launches_c1.csv python bench.py --config c1 --steps 2 --warmup 3 --no-cpu > gpurun_out/r2b_ncu_l1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_rom_solve_reg|k_rom_F_mma" -s 40 -c 2 -o gpurun_out/r2b_c3_new python tools/dev/c3_ab.py 16384 /tmp/x.npz > gpurun_out/r2b_ncu_c3.log 2>&1
echo done
