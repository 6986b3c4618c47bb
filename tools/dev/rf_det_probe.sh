# Dev probe: run-to-run determinism of the full-order solve per Rf algorithm pair
cd ${GRAFT_REPO_ROOT:-.}
for a in 1 2 3 11 12 13 21 22 23; do
  out=$(PODECM_RF_ALGS=$a timeout 200 python tools/dev/flaky_probe.py 40 2>&1)
  nz=$(echo "$out" | grep -v "^first\|^   " | awk '{print $3}' | sort -g | tail -1)
  bad=$(echo "$out" | grep -c "e-02")
  echo "algs $a: max fe-vs-first $nz, path flips $bad"
done
