"""N>1 host logic on CPU with gloo, world_size 2 (one process per "GPU"):
shard ranges, max-over-ranks timing, the row-sharded POD Gram all-reduce and
the candidate-sharded ECM argmax (identical to the single-process greedy)."""
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
