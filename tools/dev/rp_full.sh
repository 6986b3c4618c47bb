python -m pytest tests/test_gpu_rom.py tests/test_gpu_fullsize.py tests/test_gpu_rom_engines.py tests/test_gpu_twoscale.py tests/test_gpu_golden.py tests/test_gpu_pipeline.py tests/test_gpu_rom_tangent.py -q -p no:cacheprovider -x 2>&1 | tail -3
run() { python bench.py --config $2 --steps 1 --warmup 1 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); c=d['also']['$2']; print('$1', '$2', round(c.get('ms_per_step',0),1), c.get('rve_solves_per_s'), c.get('wall_s'), c.get('kernels_ms_per_step', c.get('kernels_ms')))"; }
run default c3
PODECM_ROM_CONTRACT=std run std fe2
PODECM_ROM_CONTRACT=rp run rp fe2
