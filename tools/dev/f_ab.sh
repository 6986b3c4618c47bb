set -x
python tools/dev/c3_ab.py 16384 gpurun_out/f_mma.npz > gpurun_out/f_mma.log 2>&1 || { cat gpurun_out/f_mma.log; exit 1; }
PODECM_ROM_F=fma python tools/dev/c3_ab.py 16384 gpurun_out/f_fma.npz > gpurun_out/f_fma.log 2>&1
cat gpurun_out/f_mma.log gpurun_out/f_fma.log
python -c "
import numpy as np
a=np.load('gpurun_out/f_mma.npz'); b=np.load('gpurun_out/f_fma.npz')
print('pbar rel', np.abs(a['pbar']-b['pbar']).max()/np.abs(b['pbar']).max(), 'iters equal frac', (a['iters']==b['iters']).mean(), 'status eq', np.array_equal(a['status'],b['status']))
"
python -m pytest tests/test_gpu_rom.py tests/test_gpu_fullsize.py tests/test_gpu_rom_engines.py tests/test_gpu_twoscale.py tests/test_gpu_rom_tangent.py tests/test_gpu_dropin.py -q -x 2>&1 | tail -3
