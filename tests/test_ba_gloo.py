"""World-size-2 gloo test (CPU) of the NEXT-4 global-BA sharding: keyframe
ownership as the mapping window, the sample-wide valid-ray count reduced
BEFORE any keyframe's loss is formed, then one SUM of the gradient buffer
and of the loss shares; poses rank-local."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2403_11247_b200.ba import BAStep, ba_loss_value
from paper_2403_11247_b200.window import shard

N_KF, N_G = 11, 97


def kf_count(k):
    return 3 * k + 1


def kf_contrib(k, n_valid):
    """Stand-in for one keyframe's loss + bwd: depends on the global count."""
    r = np.random.default_rng(500 + k)
    g = torch.tensor(r.standard_normal(15 * N_G + 8) / n_valid, dtype=torch.float64)
    l3 = torch.tensor([k / n_valid, 2.0 * k / n_valid, 0.01 * k], dtype=torch.float64)
    return g, l3, torch.tensor(r.standard_normal(6), dtype=torch.float64)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(rank, world):
    flat = torch.zeros(15 * N_G + 8, dtype=torch.float64)
    n_valid = torch.zeros(1, dtype=torch.int64)
    loss3 = torch.zeros(3, dtype=torch.float64)
    seen_nv = []

    def count(k):
        n_valid.add_(kf_count(k))

    def render(k, pose):
        nv = int(n_valid.item())
        seen_nv.append(nv)
        g, l3, p = kf_contrib(k, nv)
        flat.add_(g)
        loss3.add_(l3)
        pose.copy_(p)

    ba = BAStep(N_KF, flat, n_valid, loss3, count, render, rank=rank, world=world)
    out = ba.run()
    return out.clone().numpy(), loss3.clone().numpy(), seen_nv, {k: v.numpy().copy()
                                                                  for k, v in ba.poses.items()}


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    flat, l3, nv, poses = _run(rank, world)
    q.put(dict(rank=rank, flat=flat, l3=l3, nv=nv, poses=poses))
    dist.destroy_process_group()


def test_ba_world2_matches_world1():
    ref_flat, ref_l3, ref_nv, ref_poses = _run(0, 1)
    total = sum(kf_count(k) for k in range(N_KF))
    assert set(ref_nv) == {total}
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
    for r in res:
        # every keyframe's loss saw the sample-wide count, not the rank's share
        assert set(r["nv"]) == {total}
        assert np.allclose(r["flat"], ref_flat, rtol=1e-12, atol=1e-14)
        assert np.allclose(r["l3"], ref_l3, rtol=1e-12)
        assert ba_loss_value(r["l3"]) == ba_loss_value(ref_l3) or \
            abs(ba_loss_value(r["l3"]) - ba_loss_value(ref_l3)) < 1e-12
        assert sorted(r["poses"]) == shard(N_KF, r["rank"], 2)
        for k, p in r["poses"].items():
            assert np.array_equal(p, ref_poses[k])
