python tools/dev/c3_ab.py 16384 gpurun_out/tail.npz > gpurun_out/tail.log 2>&1 || { cat gpurun_out/tail.log; exit 1; }
cat gpurun_out/tail.log
python -c "
import numpy as np
a=np.load('tmp_rw_ref.npz'); b=np.load('gpurun_out/tail.npz')
for k in a: print(k, np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)))
print('pbar rel', np.abs(a['pbar']-b['pbar']).max()/np.abs(a['pbar']).max(), 'iters eq frac', (a['iters']==b['iters']).mean())
"
python -m pytest tests/test_gpu_rom.py tests/test_gpu_rom_engines.py tests/test_gpu_rom_tangent.py tests/test_gpu_twoscale.py -q -x 2>&1 | tail -2
