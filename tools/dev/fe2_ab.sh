python -m pytest tests/test_gpu_twoscale.py tests/test_gpu_rom_engines.py -q -x 2>&1 | tail -2
python bench.py --config fe2 --steps 1 --warmup 1 --no-cpu > gpurun_out/fe2.json 2> gpurun_out/fe2.err; echo "bench rc $?"
python -c "import json; d=json.load(open('gpurun_out/fe2.json')); c=d['also']['fe2']; print({k: c[k] for k in ('wall_s','macro_newton_iters','micro_evals','residual_displacement','launches')})"
