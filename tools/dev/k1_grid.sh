for m in 7 14 28 56 64 112 224 448; do
PODECM_K1_GRID_MULT=$m python bench.py --config c1 --steps 20 --warmup 5 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('mult $m', round(d['ms_per_step'],4), round(d['value']/1e9,3))"
done
