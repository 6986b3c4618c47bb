"""The split config-4 path of SURVEY §8(e) on the device: two processes (one
CUDA context each, both on cuda:0 here — the box has one GPU; their kernels
never wait on each other, every exchange is a host-side gloo collective)
run the row-sharded POD (api.pod_sharded: the DMMA Gram fused with its
reduce-scatter over CUDA-IPC peer memory — bitwise equal to the local-Gram +
all-reduce path — gathered MGS) and the candidate-sharded greedy (api.ecm_select_sharded ->
podecm_ecm_select_sharded).  Eigenvalues within 1e-12 of the single-process
POD, modes within 1e-10 up to sign, and the selected ids, iteration count and
weights equal to the single-process greedy (direct scoring), on a reduced
config-4 analogue and on a weight-drop case."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _mats():
    from paper_2307_16894_b200.api import inclusion_params, matrix_params
    return [matrix_params(), inclusion_params()]


def _inputs(api, rve, torch):
    from paper_2307_16894_b200 import synth
    U = synth.c4_snapshots(rve.export(), L=160, n_terms=6, kmax=4, seed=5, xp=torch, device=torch.device("cuda:0"))
    return U


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(__file__))
        from paper_2307_16894_b200 import api, shard
        from test_gpu_ecm_drop import _case
        torch.cuda.set_device(0)
        rve = api.Rve(32, _mats())
        U = _inputs(api, rve, torch)
        d0, d1 = shard.shard_range(U.shape[1], rank, world)
        modes, ev = api.pod_sharded(U[:, d0:d1].contiguous(), 12)  # peer-memory Gram exchange
        modes_c, ev_c = api.pod_sharded(U[:, d0:d1].contiguous(), 12, exchange="collective")
        W, _ = api.ecm_stress_snapshots(rve, U)
        H = api.ecm_mode_grads(rve, modes)
        q0, q1 = shard.shard_range(rve.n_qp, rank, world)
        opts = api.EcmOpts(eps=1e-8, max_points=60, stop_at_count=True)
        r1 = api.ecm_select_sharded(rve, H[q0:q1].contiguous(), W[:, q0:q1].contiguous(), q0, opts)
        g = api.Rve(8, _mats())
        Hd, Wd = _case(0, 0, g.n_qp)
        a0, a1 = shard.shard_range(g.n_qp, rank, world)
        T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        r2 = api.ecm_select_sharded(g, T(Hd[a0:a1]), T(Wd[:, a0:a1]), a0,
                                    api.EcmOpts(eps=1e-6, max_points=60, stop_at_count=True))
        q.put((rank, {"modes": modes.cpu().numpy(), "ev": ev.cpu().numpy(), "ecm": r1, "drop": r2,
                      "modes_c": modes_c.cpu().numpy(), "ev_c": ev_c.cpu().numpy()}))
    except Exception as e:  # surface it in the parent
        q.put((rank, {"error": repr(e)}))
    finally:
        dist.destroy_process_group()


def test_two_rank_split_config4(monkeypatch):
    import torch
    from paper_2307_16894_b200 import api
    from test_gpu_ecm_drop import _case
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=600) for _ in ps)
    for p in ps:
        p.join(timeout=120)
    for r in range(2):
        assert "error" not in res[r], res[r]
    # single-process references (direct scoring, like the sharded greedy)
    monkeypatch.setenv("PODECM_ECM_SCORE", "direct")
    rve = api.Rve(32, _mats())
    U = _inputs(api, rve, torch)
    modes, ev = api.pod(U, 12)
    W, _ = api.ecm_stress_snapshots(rve, U)
    H = api.ecm_mode_grads(rve, modes)
    ref = api.ecm_select(rve, H, W, api.EcmOpts(eps=1e-8, max_points=60, stop_at_count=True))
    g = api.Rve(8, _mats())
    Hd, Wd = _case(0, 0, g.n_qp)
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
    ref2 = api.ecm_select(g, T(Hd), T(Wd), api.EcmOpts(eps=1e-6, max_points=60, stop_at_count=True))
    ev = ev.cpu().numpy()[:12]
    m0 = modes.cpu().numpy()
    for r in range(2):
        d = res[r]
        # the peer-memory Gram exchange (GEMM fused with its reduce-scatter,
        # rank-order sums) gives the collective all-reduce's bits at 2 ranks
        assert np.array_equal(d["ev"].view(np.int64), d["ev_c"].view(np.int64))
        assert np.array_equal(d["modes"].view(np.int64), d["modes_c"].view(np.int64))
        assert np.abs(d["ev"][:12] - ev).max() <= 1e-12 * ev[0]
        sgn = np.sign((d["modes"] * m0).sum(1))
        assert np.abs(d["modes"] * sgn[:, None] - m0).max() <= 1e-10 * np.abs(m0).max()
        for got, want in ((d["ecm"], ref), (d["drop"], ref2)):
            print(f"rank {r}: ids equal {np.array_equal(got[0], want[0])}, iters {got[3]} vs {want[3]}")
            assert np.array_equal(got[0], want[0]) and got[3] == want[3]
            assert np.abs(got[1] - want[1]).max() <= 1e-9 * np.abs(want[1]).max()


def test_bench_two_rank_config4_full_size():
    """bench.py's own N=2 path at the full config-4 size (4000 snapshots,
    65,536 candidates, 400 points): re-executed under torch.distributed.run,
    both ranks on cuda:0 with gloo exchanges (PODECM_BENCH_SAME_GPU=1, the
    one-GPU stand-in for the NCCL launch); the selected ids equal the CPU
    oracle's full-size golden selection."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, PODECM_BENCH_SAME_GPU="1")
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--config", "c4", "--steps", "1",
                        "--warmup", "3", "--no-cpu"], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][-1])
    c4 = line["also"]["c4"]
    assert line["n_gpus"] == 2 and c4["selected"] == 400
    assert c4["ids_equal_golden"] is True
