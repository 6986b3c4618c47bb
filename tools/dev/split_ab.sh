python -m pytest tests/test_gpu_assembly.py tests/test_gpu_fullsize.py -q -x -k "not config3 and not config4" 2>&1 | tail -2
for sp in 1 0; do
PODECM_ASM_SPLIT=$sp python bench.py --config c2 --steps 5 --warmup 2 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['also']['c2']; print('split $sp', c['ms_per_step'], c['kernels_ms_per_step'])"
done
