"""Multi-process CPU test (gloo, world size 2) of the data-parallel plumbing: view
partition, the flat gradient layout and the single all-reduce.  Each rank computes the
oracle gradient of ITS views into a flat buffer with the product's layout; after the
all-reduce every rank must hold the gradient of all views computed in one process (the
linearity that makes views-DP exact, Q30)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2409_06765_b200 import dist as D


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _scene():
    from synth import scenes as S
    return S.tiny_scene(9, N=60, width=48, height=40, sh_degree=1, views=4)


def _grads_for(sc, views, o, v_img):
    import oracle
    s = dict(sc)
    s["viewmats"] = sc["viewmats"][views]
    s["Ks"] = sc["Ks"][views]
    return oracle.forward_backward(s, o, v_img[views], with_isect=False)["grads"]


def _fill_flat(g, N, K):
    _, total = D.flat_layout(N, K, True)
    flat = torch.zeros(total, dtype=torch.float64)
    v = D.views(flat, N, K, True)
    v["quats"].copy_(torch.from_numpy(g["v_quats"]))
    v["means"].copy_(torch.from_numpy(g["v_means"]))
    v["scales"].copy_(torch.from_numpy(g["v_scales"]))
    v["opacities"].copy_(torch.from_numpy(g["v_opacities"]))
    v["colors"].copy_(torch.from_numpy(g["v_colors"]))
    return flat


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    sc = _scene()
    o = oracle.Options(sh_degree=1)
    rng = np.random.default_rng(0)
    v_img = rng.normal(size=(4, 40, 48, 3))
    mine = D.partition_views(4, world, rank)
    g = _grads_for(sc, mine, o, v_img)
    flat = _fill_flat(g, 60, 4)
    D.allreduce_grads(flat)
    q.put((rank, mine, flat.numpy()))
    dist.destroy_process_group()


def test_partition_views_covers_all_contiguously():
    for V in [1, 4, 8, 32]:
        for R in [1, 2, 4, 8]:
            parts = [D.partition_views(V, R, r) for r in range(R)]
            assert sorted(sum(parts, [])) == list(range(V))
            for p in parts:
                assert p == list(range(p[0], p[0] + len(p))) if p else True


def test_flat_layout_aligned_and_disjoint():
    lay, total = D.flat_layout(1001, 16, True)
    end = 0
    for name, (off, n, shp) in lay.items():
        assert off % 4 == 0 and off >= end
        assert int(np.prod(shp)) == n
        end = off + n
    assert total >= end


def test_gloo_allreduce_equals_single_process():
    import oracle
    oracle.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sc = _scene()
    o = oracle.Options(sh_degree=1)
    v_img = np.random.default_rng(0).normal(size=(4, 40, 48, 3))
    ref = _fill_flat(_grads_for(sc, [0, 1, 2, 3], o, v_img), 60, 4).numpy()
    assert sorted(sum([r[1] for r in res], [])) == [0, 1, 2, 3]
    for _, _, flat in res:
        np.testing.assert_allclose(flat, ref, rtol=1e-12, atol=1e-15)
