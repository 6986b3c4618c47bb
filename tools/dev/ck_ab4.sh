python tools/dev/c3_ab.py 16384 gpurun_out/yf_base.npz > gpurun_out/yf_base.log 2>&1 || { cat gpurun_out/yf_base.log; exit 1; }
PODECM_ROM_CHECK_IPW=4 python tools/dev/c3_ab.py 16384 gpurun_out/yf.npz > gpurun_out/yf.log 2>&1 || { cat gpurun_out/yf.log; exit 1; }
cat gpurun_out/yf_base.log gpurun_out/yf.log
python -c "
import numpy as np
a=np.load('gpurun_out/yf_base.npz'); b=np.load('gpurun_out/yf.npz')
for k in a: print(k, np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)))
print('pbar rel', np.abs(a['pbar']-b['pbar']).max()/np.abs(a['pbar']).max(), 'iters eq', (a['iters']==b['iters']).mean())
"
