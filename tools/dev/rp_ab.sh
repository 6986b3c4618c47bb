python -m pytest tests/test_gpu_rom.py tests/test_gpu_fullsize.py -q -p no:cacheprovider -k "not config2 and not config4" 2>&1 | tail -1
run() { python bench.py --config c3 --steps 1 --warmup 1 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); c=d['also']['c3']; print('$1', 'c3 ms', round(c['ms_per_step'],1), round(c['rve_solves_per_s']), c['kernels_ms_per_step']['k_rom_contract'], c['failed_instances'])"; }
PODECM_ROM_CONTRACT=rp23 run rp23
run rp33
