python tools/dev/pod_debug.py > gpurun_out/plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_eig_cholinv -s 5 -c 1 -o gpurun_out/r2_cholinv python tools/dev/pod_debug.py > gpurun_out/ncu.log 2>&1
echo rc $?
