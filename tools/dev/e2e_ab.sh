python - <<'PY'
import torch, time
d=torch.empty(872*2**20//8, dtype=torch.float64, device='cuda'); h=torch.empty_like(d, device='cpu').pin_memory()
d2=torch.empty(335*2**20//8, dtype=torch.float64, device='cuda'); h2=torch.empty_like(d2, device='cpu').pin_memory()
s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
for name,fn in [("d2h",lambda: h.copy_(d,non_blocking=True)),("h2d",lambda: d2.copy_(h2,non_blocking=True))]:
    for _ in range(2): fn()
    torch.cuda.synchronize(); t=time.perf_counter()
    for _ in range(5): fn()
    torch.cuda.synchronize(); dt=(time.perf_counter()-t)/5
    print(name, "ms", round(dt*1e3,2))
torch.cuda.synchronize(); t=time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): h.copy_(d,non_blocking=True)
    with torch.cuda.stream(s2): d2.copy_(h2,non_blocking=True)
torch.cuda.synchronize(); print("both ms", round((time.perf_counter()-t)/5*1e3,2))
PY
for cfg in "8 3" "4 3" "16 3" "16 4" "32 4" "8 2"; do set -- $cfg
PODECM_E2E_CHUNKS=$1 PODECM_E2E_STREAMS=$2 python bench.py --config c1 --steps 10 --warmup 3 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('chunks $1 streams $2 e2e', round(d['e2e']['value']/1e6,1), 'M pts/s')"
done
