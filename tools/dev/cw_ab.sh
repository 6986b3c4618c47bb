python tools/dev/c3_ab.py 16384 gpurun_out/rw.npz > gpurun_out/rw.log 2>&1 || { cat gpurun_out/rw.log; exit 1; }
PODECM_ROM_CONTRACT=cw python tools/dev/c3_ab.py 16384 gpurun_out/cw.npz > gpurun_out/cw.log 2>&1 || { cat gpurun_out/cw.log; exit 1; }
cat gpurun_out/rw.log gpurun_out/cw.log
python -c "
import numpy as np
a=np.load('gpurun_out/rw.npz'); b=np.load('gpurun_out/cw.npz')
for k in a: print(k, np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)))
"
