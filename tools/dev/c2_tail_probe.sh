python -m pytest tests/test_gpu_assembly.py -q -p no:cacheprovider 2>&1 | tail -2
run() { python bench.py --config c2 --steps 5 --warmup 2 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); c=d['also']['c2']; print('$1', 'c2 ms', round(c['ms_per_step'],3), c['kernels_ms_per_step'], 'c0', d['also'].get('c0',{}).get('ms_per_step'))"; }
run staged
