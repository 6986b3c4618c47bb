set -x
python tools/dev/c3_ab.py 16384 gpurun_out/lu_reg.npz > gpurun_out/lu_reg.log 2>&1 || { cat gpurun_out/lu_reg.log; exit 1; }
PODECM_ROM_LU=smem python tools/dev/c3_ab.py 16384 gpurun_out/lu_smem.npz > gpurun_out/lu_smem.log 2>&1
cat gpurun_out/lu_reg.log gpurun_out/lu_smem.log
python -c "
import numpy as np
a=np.load('gpurun_out/lu_reg.npz'); b=np.load('gpurun_out/lu_smem.npz')
for k in a: print(k, np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)))
"
python -m pytest tests/test_gpu_rom.py tests/test_gpu_fullsize.py tests/test_gpu_rom_engines.py tests/test_gpu_twoscale.py -q -x 2>&1 | tail -3
