#!/bin/bash
# A/B prebuilt library variants paper_2307_16894_b200/var_<name>.so on config 3
cd ${GRAFT_REPO_ROOT:-.}
L=paper_2307_16894_b200/libpodecm_cuda.so
for v in ${VARIANTS}; do
  cp paper_2307_16894_b200/var_$v.so $L
  timeout 300 python -m pytest tests/test_gpu_rom.py tests/test_gpu_golden.py -x -q 2>&1 | tail -1 | sed "s/^/$v tests: /"
  python bench.py --config ${CFG:-c3} --c3-inst ${C3N:-16384} --steps 1 --warmup 1 --no-cpu > gpurun_out/ab_$v.json 2> gpurun_out/ab_$v.err
  python -c "import json; d=json.load(open('gpurun_out/ab_$v.json')); c=d['also']['c3']; print('$v', round(c['ms_per_step'],1), c['kernels_ms_per_step'], c['failed_instances'])" || tail -3 gpurun_out/ab_$v.err
done
cp paper_2307_16894_b200/var_base.so $L
