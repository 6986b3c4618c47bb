python -m pytest tests/test_gpu_rom.py tests/test_gpu_fullsize.py tests/test_gpu_rom_engines.py tests/test_gpu_twoscale.py tests/test_gpu_golden.py tests/test_gpu_pipeline.py tests/test_gpu_rom_tangent.py -q -p no:cacheprovider 2>&1 | tail -15 > gpurun_out/rp_tests.log; tail -2 gpurun_out/rp_tests.log
for tr in 0.075 0.05; do for m in std rp; do
PODECM_FE2_TRACTION=$tr PODECM_ROM_CONTRACT=$m python bench.py --config fe2 --steps 1 --warmup 1 --no-cpu 2>/dev/null | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.readlines()[-1]); c=d['also']['fe2']; print('$tr $m', c.get('wall_s'), c.get('error','')[:80], (c.get('kernels_ms') or {}).get('k_rom_contract'))
except Exception as e: print('$tr $m fail', e)"
done; done
