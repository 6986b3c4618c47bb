run() { python bench.py --config c3 --c3-inst ${C3N:-16384} --steps 1 --warmup 1 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); c=d['also']['c3']; print('$1', 'c3 ms', round(c['ms_per_step'],1), round(c['rve_solves_per_s']), c['kernels_ms_per_step']['k_rom_contract'], c['failed_instances'])"; }
PODECM_ROM_CONTRACT=std run std
for v in 0; do
PODECM_ROM_CONTRACT=rp PODECM_ROM_RP_VAR=$v python -m pytest tests/test_gpu_rom.py -q -p no:cacheprovider -k "remainder_packed" -s 2>&1 | grep -E "rp vs std|passed|failed"
PODECM_ROM_RP_VAR=$v run rp$v; done
