# round-2 evidence: plain runs first (exit 0), then the ncu captures
set -x
python bench.py --config c1 --steps 3 --warmup 3 --no-cpu > gpurun_out/plain_c1.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r2_launches_c1.csv python bench.py --config c1 --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_l1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_material --launch-skip 3 --launch-count 1 -o gpurun_out/r2_c1_material_final python bench.py --config c1 --steps 3 --warmup 3 --no-cpu > gpurun_out/ncu_c1.log 2>&1
python bench.py --config c2 --c2-inst 128 --steps 1 --warmup 1 --no-cpu > gpurun_out/plain_c2.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_asm_qp2|k_asm_gather" --launch-skip 2 --launch-count 2 -o gpurun_out/r2_c2_asm python bench.py --config c2 --c2-inst 128 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_c2.log 2>&1
python tools/dev/pod_debug.py > gpurun_out/plain_pod.log 2>&1 || exit 1
ncu --set full --clock-control none -k regex:"k_eig|k_gemm_dmma|k_mgs" --launch-skip 40 --launch-count 6 -o gpurun_out/r2_pod python tools/dev/pod_debug.py > gpurun_out/ncu_pod.log 2>&1
echo done
