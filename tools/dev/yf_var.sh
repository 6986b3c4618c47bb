for v in 0 1 2 3 4 5; do
PODECM_ROM_CONTRACT=yf PODECM_YF_V=$v python tools/dev/c3_ab.py 16384 gpurun_out/yf_$v.npz 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('v$v', d['kernels_ms']['k_rom_contract'])"
done
python tools/dev/c3_ab.py 16384 gpurun_out/yf_base.npz 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('base', d['kernels_ms']['k_rom_contract'])"
python -c "
import numpy as np
a=np.load('gpurun_out/yf_base.npz')
for v in range(6):
    b=np.load(f'gpurun_out/yf_{v}.npz'); print(v, all(np.array_equal(a[k].view(np.uint8), b[k].view(np.uint8)) for k in a))
"
