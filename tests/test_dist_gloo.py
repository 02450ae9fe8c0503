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


# ---- Gaussian-sharded exchange (NEXT-4(i), paper_2409_06765_b200.gshard) ----------------
def _shard_worker(rank, world, port, q, n_views):
    """Each rank plays the owner of a shard with camera-major items and the renderer of its
    views: rows encode (source rank, camera, local item); the forward all-to-all must deliver
    exactly the rows of the renderer's cameras, source rank-major, in each source's order,
    and the backward all-to-all must return every row to the position it came from."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2409_06765_b200 import gshard as G
    vs = G.view_starts(n_views, world)
    rng = np.random.default_rng(100 + rank)
    per_cam = rng.integers(0, 7, size=n_views)          # items per camera on this owner
    cams = np.repeat(np.arange(n_views), per_cam)       # camera-major (gs_project_packed order)
    n = cams.size
    send = torch.zeros((n, 16), dtype=torch.float32)
    send[:, 0] = rank
    send[:, 1] = torch.from_numpy(cams.astype(np.float32))
    send[:, 2] = torch.arange(n, dtype=torch.float32)
    counts = torch.tensor([int(((cams >= vs[d]) & (cams < vs[d + 1])).sum()) for d in range(world)],
                          dtype=torch.int64)
    ex = G.Exchange()
    assert ex.world == world
    recv_counts = ex.counts(counts)
    rs, ss = recv_counts.tolist(), counts.tolist()
    recv = torch.zeros((sum(rs), 16), dtype=torch.float32)
    ex.rows(recv, send, rs, ss)
    # "render": tag every received row, then send it back
    back_in = recv.clone()
    back_in[:, 3] = 1000 + rank
    back = torch.zeros_like(send)
    ex.rows(back, back_in, ss, rs)
    q.put((rank, vs, cams, recv.numpy(), rs, back.numpy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n_views", [(2, 4), (3, 2), (3, 7)])
def test_gloo_sharded_exchange_routing(world, n_views):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, q, n_views)) for r in range(world)]
    for p in procs:
        p.start()
    res = {r[0]: r[1:] for r in (q.get(timeout=300) for _ in range(world))}
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    vs = res[0][0]
    for d in range(world):
        _, _, recv, rs, _ = res[d]
        # expected: for each source rank in order, its items of cameras [vs[d], vs[d+1]) in order
        exp = []
        for s in range(world):
            cams = res[s][1]
            idx = np.nonzero((cams >= vs[d]) & (cams < vs[d + 1]))[0]
            exp += [(s, cams[i], i) for i in idx]
            assert rs[s] == idx.size
        got = [(int(r[0]), int(r[1]), int(r[2])) for r in recv]
        assert got == exp
    for s in range(world):
        _, cams, _, _, back = res[s]
        assert np.array_equal(back[:, 0], np.full(cams.size, s))
        assert np.array_equal(back[:, 2], np.arange(cams.size))            # back in place
        owner = np.searchsorted(vs, cams, side="right") - 1                 # renderer of each item
        assert np.array_equal(back[:, 3], 1000 + owner)


def test_view_starts_and_shards():
    from paper_2409_06765_b200 import gshard as G
    for V in [1, 2, 5, 32]:
        for R in [1, 2, 3, 8]:
            vs = G.view_starts(V, R)
            assert vs[0] == 0 and vs[-1] == V and all(a <= b for a, b in zip(vs, vs[1:]))
            for r in range(R):
                assert list(range(vs[r], vs[r + 1])) == D.partition_views(V, R, r)
            rng = [G.shard_range(1001, R, r) for r in range(R)]
            assert rng[0][0] == 0 and rng[-1][1] == 1001
            assert all(a[1] == b[0] for a, b in zip(rng, rng[1:]))


def test_exchange_world1_and_distributed_api_validation():
    """Host logic without a process group: the world-size-1 exchange degenerates to copies,
    and rasterization(distributed=True) rejects the options it does not combine with."""
    from paper_2409_06765_b200 import gshard as G
    ex = G.Exchange()
    assert ex.world == 1
    c = torch.tensor([5], dtype=torch.int64)
    assert ex.counts(c).tolist() == [5]
    src = torch.arange(10, dtype=torch.float32).reshape(5, 2)
    dst = torch.zeros_like(src)
    ex.rows(dst, src, [5], [5])
    assert torch.equal(dst, src)
    from paper_2409_06765_b200 import rasterization
    z = torch.zeros
    args = (z(4, 3), z(4, 4), z(4, 3), z(4), z(4, 3), z(1, 4, 4), z(1, 3, 3), 16, 16)
    with pytest.raises(ValueError):
        rasterization(*args, distributed=True, render_mode="RGB+D")
    with pytest.raises(ValueError):
        rasterization(*args, distributed=True, absgrad=True)


def test_bucket_layout_covers_every_gaussian_once():
    """dist.bucket_layout: buckets tile [0, N) in order with 128-aligned starts, every section
    16-byte aligned, one contiguous slice per bucket; gather_buckets inverts bucket_views."""
    for N, nb in [(1000, 4), (20000, 3), (130, 8), (0, 4), (128, 1)]:
        lay, total = D.bucket_layout(N, 16, True, nb)
        n = 0
        for n0, n1, off, secs in lay:
            assert n0 == n and n0 % 128 == 0 and n1 >= n0
            n = n1
            for o, s, shp in secs.values():
                assert o % 4 == 0 and off <= o and o + s <= total
        assert n == N
        flat = torch.arange(total, dtype=torch.float32)
        vs = D.bucket_views(flat, lay)
        g = D.gather_buckets(flat, lay)
        assert g["means"].shape == (N, 3) and g["colors"].shape == (N, 16, 3) and g["quats"].shape == (N, 4)
        for v in vs:
            assert torch.equal(g["means"][v["n0"]:v["n1"]], v["means"])
            assert v["flat"].data_ptr() <= v["means"].data_ptr()
        # sections never overlap: every float index used at most once
        used = torch.cat([t.reshape(-1) for v in vs for k, t in v.items() if k not in ("n0", "n1", "flat")])
        assert used.unique().numel() == used.numel()
