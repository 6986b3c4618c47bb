#!/bin/bash
# A/B environment-variable variants of the library on one bench config.
#   CASES="name1:VAR=a,VAR2=b name2:VAR=c" CFG=c2 TESTS="tests/test_gpu_assembly.py" bash tools/ab_env.sh
cd ${GRAFT_REPO_ROOT:-.}
for cs in ${CASES}; do
  name=${cs%%:*}; envs=${cs#*:}
  envline=$(echo "$envs" | tr ',' ' ')
  if [ -n "$TESTS" ]; then
    env $envline timeout 600 python -m pytest $TESTS -x -q 2>&1 | tail -1 | sed "s/^/$name tests: /"
  fi
  env $envline python bench.py --config ${CFG} ${BENCH_ARGS} --no-cpu > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err
  python - "$name" "$CFG" <<'PY'
import json, sys
name, cfg = sys.argv[1], sys.argv[2]
d = json.load(open(f"gpurun_out/ab_{name}.json"))
c = d["also"].get(cfg) if cfg != "c1" else d
keep = {k: v for k, v in c.items() if k in ("ms_per_step", "kernels_ms_per_step", "qp_per_s", "rve_solves_per_s", "failed_instances", "value")}
print(name, keep)
PY
done
