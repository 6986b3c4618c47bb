# round-2 (session 4) evidence refresh: tests, smoke, full bench, reference arm
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2c_gputest.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/r2c_gputest.log
python __graft_entry__.py --smoke > gpurun_out/r2c_smoke.log 2>&1; echo "smoke rc $?"; tail -1 gpurun_out/r2c_smoke.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2c_bench_all.json 2> gpurun_out/r2c_bench_all.err; echo "bench rc $?"
python -c "import json; d=json.loads(open('gpurun_out/r2c_bench_all.json').read().strip().splitlines()[-1]); print(json.dumps(d['baseline_metrics']))"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2c_bench_ref.json 2>&1; echo "ref rc $?"; tail -c 600 gpurun_out/r2c_bench_ref.json
echo done
