# C1 variant A/B: bitwise tests on the default, then bench timings per variant
python -m pytest tests/test_gpu_material_fullscale.py tests/test_gpu_material.py -q -x 2>&1 | tail -2
for v in ${K1V:-5 7}; do
  PODECM_K1_VARIANT=$v python bench.py --config c1 --steps 20 --warmup 5 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('variant $v', d['ms_per_step'], d['roofline']['kernel_ms'])"
done
