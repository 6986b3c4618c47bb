#!/bin/bash
# two ranks on the one GPU of a gpurun box (gloo exchanges): the sharded C4 bench path end to end
cd "$(dirname "$0")/../.."
mkdir -p gpurun_out
PODECM_BENCH_SAME_GPU=1 timeout 600 python bench.py --gpus 2 --config c4 --steps 1 --warmup 3 --no-cpu > gpurun_out/c4_2rank.log 2> gpurun_out/c4_2rank.err
echo rc=$?
tail -3 gpurun_out/c4_2rank.err
python - <<'P'
import json
l=[x for x in open("gpurun_out/c4_2rank.log") if x.startswith("{")]
d=json.loads(l[-1]); c=d.get("also",{}).get("c4",d)
print({k:c.get(k) for k in ("ms_per_step","selected","ids_equal_golden","ecm_residual_rel","split","pod_stage_s","ecm_greedy_s")})
P
