cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
A="--config c3 --c3-inst 65536 --steps 1 --warmup 1 --no-cpu"
run() { python bench.py $A > gpurun_out/ab_$1.json 2>gpurun_out/ab_$1.err; python -c "
import json;d=json.load(open('gpurun_out/ab_$1.json'));c=d['also']['c3'];print('$1',round(c['ms_per_step'],1),c['kernels_ms_per_step'])"; }
PODECM_ROM_LAZY=0 run fused1
PODECM_ROM_LAZY=1 run lazy1
cp paper_2307_16894_b200/libpodecm_cuda.so /tmp/new.so; cp build/libpodecm_old.so paper_2307_16894_b200/libpodecm_cuda.so
run old1
cp /tmp/new.so paper_2307_16894_b200/libpodecm_cuda.so
PODECM_ROM_LAZY=0 run fused2
