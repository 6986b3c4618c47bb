python -m pytest tests/test_gpu_rom.py -q -p no:cacheprovider 2>&1 | tail -1
python bench.py --config c3 --steps 2 --warmup 1 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); c=d['also']['c3']; print('c3 solves/s', round(d['value']), 'ms', round(c['ms_per_step'],1), c['kernels_ms_per_step'])"
