for m in 4 5 6; do
PODECM_ASM_EMINB=$m python bench.py --config c2 --steps 5 --warmup 2 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); c=d['also']['c2']; print('eminb $m', c['ms_per_step'], c['kernels_ms_per_step'])"
done
python bench.py --config c2 --c2-inst 128 --steps 1 --warmup 1 --no-cpu > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_asm_qp2" --launch-skip 2 --launch-count 1 -o gpurun_out/r2b_c2split python bench.py --config c2 --c2-inst 128 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_c2s.log 2>&1
