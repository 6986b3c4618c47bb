cd ${GRAFT_REPO_ROOT:-.}
L=paper_2307_16894_b200/libpodecm_cuda.so
for v in ${VARIANTS}; do
  cp paper_2307_16894_b200/var_$v.so $L
  for k in ${K1V:-5}; do
  PODECM_K1_VARIANT=$k python bench.py --config c1 --steps 20 --warmup 5 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v k1v=$k', d['ms_per_step'], d['roofline']['kernel_ms'])"
  done
done
cp paper_2307_16894_b200/var_base.so $L
