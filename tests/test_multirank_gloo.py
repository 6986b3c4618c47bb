"""N>1 host logic on CPU with gloo, world_size 2 (one process per "GPU"):
shard ranges, max-over-ranks timing, the row-sharded POD Gram all-reduce,
the candidate-sharded ECM argmax, the whole candidate-sharded greedy (the
device path's algorithm, oracle/pod_ecm.ecm_select_sharded: ids identical to
the single-rank greedy, weight drops included) and the bench launcher
(`bench.py --gpus 2` re-executing itself under torch.distributed.run)."""
import os
import socket

import numpy as np
import torch.multiprocessing as mp

from paper_2307_16894_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out = {}
        # timing: max over ranks
        out["max"] = shard.max_over_ranks(float(rank + 1))
        # Gram of a row-sharded snapshot matrix
        rng = np.random.default_rng(0)
        S = rng.standard_normal((1003, 37))
        lo, hi = shard.shard_range(S.shape[0], rank, world)
        g = torch.from_numpy(S[lo:hi].T @ S[lo:hi])
        shard.allreduce_gram(g)
        out["gram_err"] = float(np.abs(g.numpy() - S.T @ S).max())
        # candidate-sharded argmax with a tie across the shard boundary
        scores = rng.uniform(0, 1, 101)
        scores[10] = scores[70] = 2.0  # tie: smallest index (10) must win
        lo, hi = shard.shard_range(len(scores), rank, world)
        loc = scores[lo:hi]
        k = int(np.argmax(loc))
        s, i = shard.argmax_over_ranks(float(loc[k]), lo + k)
        out["argmax"] = (s, i)
        # the candidate-sharded greedy: a C4-like case and a weight-drop case
        from oracle import pod_ecm
        import sys
        sys.path.insert(0, os.path.dirname(__file__))
        from test_gpu_ecm_drop import _case
        nq = 256
        wq = np.random.default_rng(3).uniform(0.5, 1.5, nq) / nq
        out["greedy"] = []
        for seed, power in ((0, 0), (11, None)):
            if power is None:
                r2 = np.random.default_rng(seed)
                H, W = r2.normal(size=(nq, 6, 4)), r2.normal(size=(9, nq, 4))
                kw = dict(eps=1e-9, max_points=40, stop_at_count=True)
            else:
                H, W = _case(seed, power, nq)
                kw = dict(eps=1e-6, max_points=60, stop_at_count=True)
            lo, hi = shard.shard_range(nq, rank, world)
            got = pod_ecm.ecm_select_sharded(H[lo:hi], W[:, lo:hi], wq, lo, **kw)
            st = {}
            ref = pod_ecm.ecm_select(H, W, wq, stats=st, **kw)
            out["greedy"].append((got[0].tolist(), ref[0].tolist(), got[3], ref[3],
                                  float(np.abs(got[1] - ref[1]).max()), st.get("drops", 0)))
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_shard_ranges_cover():
    for n, w in ((10, 3), (65536, 8), (5, 8)):
        rs = [shard.shard_range(n, r, w) for r in range(w)]
        assert rs[0][0] == 0 and rs[-1][1] == n
        assert all(rs[k][1] == rs[k + 1][0] for k in range(w - 1))


def test_two_rank_collectives():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(2):
        assert res[r]["max"] == 2.0
        assert res[r]["gram_err"] <= 1e-11
        assert res[r]["argmax"] == (2.0, 10)
        drops = 0
        for got_ids, ref_ids, got_it, ref_it, dw, nd in res[r]["greedy"]:
            assert got_ids == ref_ids and got_it == ref_it and dw <= 1e-10
            drops += nd
        assert drops >= 1  # the weight-drop branch ran inside the sharded greedy


def test_bench_launcher_two_ranks():
    """`bench.py --gpus 2` re-executes itself under torch.distributed.run
    (one process per GPU, 127.0.0.1 rendezvous); here with the CPU stub step
    (gloo): rank 0 prints one JSON line with n_gpus 2 and the max-over-ranks
    time."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--config", "launch-stub",
                        "--steps", "3", "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=root)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["value"] > 0
    assert d["config"]["ranks_seen"] == [0, 1]
