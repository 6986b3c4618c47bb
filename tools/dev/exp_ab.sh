L=paper_2307_16894_b200/libpodecm_cuda.so
cp $L /tmp/keep.so
for v in ${VARS}; do
  cp paper_2307_16894_b200/var_$v.so $L
  python tools/dev/c3_ab.py ${C3N:-16384} /tmp/x_$v.npz 2>&1 | tail -1 | sed "s/^/$v /"
done
cp /tmp/keep.so $L
