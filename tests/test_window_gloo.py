"""World-size-2 gloo tests (CPU) of the keyframe-window data parallelism
(SURVEY.md §8(e)): ownership, the single gradient all-reduce, rank-local pose
gradients and bit-identical replicas after a deterministic update."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_11247_b200.window import WindowStep, apply_sgd, shard

N_KF, N_G = 13, 257


def contrib(k):
    """Deterministic stand-in for one keyframe's fwd+bwd gradient."""
    r = np.random.default_rng(1000 + k)
    return (torch.tensor(r.standard_normal(15 * N_G + 8), dtype=torch.float32),
            torch.tensor(r.standard_normal(6), dtype=torch.float32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    flat = torch.zeros(15 * N_G + 8)
    rendered = []

    def render(k, pose):
        g, p = contrib(k)
        flat.add_(g)
        pose.copy_(p)
        rendered.append(k)

    prepared = []
    ws = WindowStep(N_KF, flat, render, prepare_fn=lambda: prepared.append(1))
    params = torch.linspace(-1, 1, flat.numel())
    for it in range(3):
        out = ws.run()
        apply_sgd([params], [out], lr=0.01)
    # replica check: gather the parameters of every rank
    gathered = [torch.zeros_like(params) for _ in range(world)]
    dist.all_gather(gathered, params)
    q.put(dict(rank=rank, rendered=rendered, flat=out.clone().numpy(),
               poses={k: v.numpy().copy() for k, v in ws.poses.items()},
               same=all(torch.equal(gathered[0], g) for g in gathered), prepared=len(prepared)))
    dist.destroy_process_group()


def test_shard_round_robin():
    for world in (1, 2, 4, 8):
        owned = sorted(k for r in range(world) for k in shard(64, r, world))
        assert owned == list(range(64))
        loads = [len(shard(64, r, world)) for r in range(world)]
        assert max(loads) - min(loads) <= 1
    with pytest.raises(ValueError):
        shard(4, 2, 2)


def test_window_allreduce_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort(key=lambda d: d["rank"])
    expect = sum(contrib(k)[0].double() for k in range(N_KF)).numpy()
    for r in res:
        # each rank rendered exactly its keyframes, 3 iterations
        assert sorted(set(r["rendered"])) == shard(N_KF, r["rank"], 2)
        assert len(r["rendered"]) == 3 * len(shard(N_KF, r["rank"], 2))
        assert r["prepared"] == 3
        # the reduced buffer is the sum over ALL keyframes, on both ranks
        assert np.allclose(r["flat"], expect, rtol=1e-5, atol=1e-5)
        # pose gradients stay local to the owner
        assert sorted(r["poses"]) == shard(N_KF, r["rank"], 2)
        for k, p in r["poses"].items():
            assert np.array_equal(p, contrib(k)[1].numpy())
        assert r["same"]
    assert np.array_equal(res[0]["flat"], res[1]["flat"])
