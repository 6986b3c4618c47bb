python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2_gputest.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/r2_gputest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench_all.json 2> gpurun_out/r2_bench_all.err; echo "bench rc $?"
python -c "import json; d=json.loads(open('gpurun_out/r2_bench_all.json').read().strip().splitlines()[-1]); print(json.dumps(d['baseline_metrics']))"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r2_bench_ref.json 2>&1; echo "ref rc $?"; tail -c 400 gpurun_out/r2_bench_ref.json
