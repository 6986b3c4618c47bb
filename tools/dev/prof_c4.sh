python bench.py --config c4 --steps 1 --warmup 0 --no-cpu > gpurun_out/plain_c4.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"k_ecm_gram_cols" --launch-skip 30 --launch-count 2 -o gpurun_out/r2b_c4_gram python bench.py --config c4 --steps 1 --warmup 0 --no-cpu > gpurun_out/ncu_c4.log 2>&1
echo done
