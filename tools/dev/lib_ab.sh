# A/B two prebuilt libraries (var_base.so, var_new.so) on one C3 solve, bitwise
L=paper_2307_16894_b200/libpodecm_cuda.so
cp $L /tmp/keep.so
for v in base new; do
  cp paper_2307_16894_b200/var_$v.so $L
  python tools/dev/c3_ab.py ${C3N:-16384} gpurun_out/lib_$v.npz > gpurun_out/lib_$v.log 2>&1 || cat gpurun_out/lib_$v.log
  cat gpurun_out/lib_$v.log
done
cp /tmp/keep.so $L
python -c "
import numpy as np
a=np.load('gpurun_out/lib_base.npz'); b=np.load('gpurun_out/lib_new.npz')
for k in a: print(k, np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)))
"
rm -f gpurun_out/lib_*.npz
