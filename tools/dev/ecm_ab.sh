python -m pytest tests/test_gpu_pod_ecm.py tests/test_gpu_ecm_drop.py tests/test_gpu_sharded.py -q -x 2>&1 | tail -2
python -m pytest tests/test_gpu_fullsize.py -q -x -k config4 2>&1 | tail -2
for sp in ${SPECS:-0 4 7}; do
PODECM_ECM_SPEC=$sp python bench.py --config c4 --steps 2 --warmup 1 --no-cpu > gpurun_out/c4_$sp.json 2> gpurun_out/c4_$sp.err
python -c "import json; d=json.load(open('gpurun_out/c4_$sp.json')); c=d['also']['c4']; print('spec $sp', c['ms_per_step'], c['ecm_greedy_s'], c['ids_equal_golden'], c['kernel_calls_per_step'].get('k_ecm_gram_col'), c['kernels_ms_per_step'].get('k_ecm_gram_col'))"
done
