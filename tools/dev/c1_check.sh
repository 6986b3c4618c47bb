# C1 correctness (device gm == glibc; all 2^22 points bitwise) + timing
python -m pytest tests/test_gpu_gmath.py tests/test_gpu_material_fullscale.py tests/test_gpu_material.py -q -p no:cacheprovider 2>&1 | tail -2
for v in ${K1_VARIANTS:-default}; do
  if [ "$v" != default ]; then export PODECM_K1_VARIANT=$v; fi
  python bench.py --config c1 --steps 20 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('variant', '$v', 'ms', round(d['ms_per_step'],4), 'kernel_ms', d['roofline']['kernel_ms'], 'Gpt/s', round(d['value']/1e9,3))"
done
