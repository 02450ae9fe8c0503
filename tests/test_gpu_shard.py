"""GPU parity of the Gaussian-sharded step (include/gs.h
"Gaussian-sharded scale-out").  One GPU, R simulated ranks: each rank's kernels run on its
own Gaussian shard / view block, and the all-to-all is stood in for by slicing the send
rows exactly as `all_to_all_single` would (the NCCL/gloo call itself is covered by
tests/test_dist_gloo.py).  The sharded result must equal the one-GPU call: images, T and
last splat ids bit-identical (same splats in the same order, include/gs.h), gradients of
every shard equal to the one-GPU gradients up to fp32 atomic order, and both within the
parity contract against the oracle."""
import numpy as np
import pytest

import oracle
from synth import scenes as S
from tests import parity_util as U

pytestmark = pytest.mark.gpu

PARAM_KEYS = ["means", "quats", "scales", "opacities", "colors"]
GRAD_KEYS = ["v_means", "v_quats", "v_scales", "v_opacities", "v_colors"]


def _route(engines, forward=True):
    """The all-to-all of include/gs.h, in one process: renderer q receives, source
    rank-major, rows [off_r(q), off_r(q) + send_r[q]) of every source r (forward); the
    backward returns the renderers' per-item gradients along the reversed splits."""
    import torch
    R = len(engines)
    offs = [np.concatenate([[0], np.cumsum(e.send_splits)]) for e in engines]
    if forward:
        for q, e in enumerate(engines):
            e.recv_splits = [engines[r].send_splits[q] for r in range(R)]
            e.n_recv = sum(e.recv_splits)
            if e._alloc_recv(e.n_recv + 16):
                e._alloc_isect(max(e.cap, 4 * e.rcap))
            parts = [engines[r].send[offs[r][q]:offs[r][q + 1]] for r in range(R)]
            if e.n_recv:
                e.recv[:e.n_recv].copy_(torch.cat(parts))
    else:
        for q, e in enumerate(engines):
            roff = np.concatenate([[0], np.cumsum(e.recv_splits)])
            for r in range(R):
                engines[r].v_splats[offs[r][q]:offs[r][q + 1]].copy_(e.r_v_splats[roff[r]:roff[r + 1]])


def run_sharded(sc, R, v_img, antialiased=False, nnz_capacity=None):
    import torch
    from paper_2409_06765_b200.gshard import ShardedEngine, shard_range
    C, N = sc["viewmats"].shape[0], sc["means"].shape[0]
    W, H, deg = int(sc["width"]), int(sc["height"]), int(sc["sh_degree"])
    K = sc["colors"].shape[1] if deg >= 0 else None
    full = U.to_torch(sc, "cuda")
    engines, params = [], []
    for r in range(R):
        n0, n1 = shard_range(N, R, r)
        engines.append(ShardedEngine(n1 - n0, C, W, H, rank=r, world=R, sh_degree=deg, K=K, antialiased=antialiased,
                                     nnz_capacity=nnz_capacity, M_capacity=64 if nnz_capacity else None))
        params.append(tuple(t[n0:n1].contiguous() for t in full[:5]) + full[5:])
    for e, p in zip(engines, params):
        while True:
            e.project_and_pack(*p)
            if e.read_send_counts():
                break
    _route(engines, forward=True)
    v = torch.from_numpy(np.ascontiguousarray(v_img, np.float32)).cuda()
    for e in engines:
        while True:
            e.render_forward()
            if not e.check_isect_capacity():
                break
        e.render_backward(v[e.c0:e.c1].contiguous() if e.C_loc else None)
    _route(engines, forward=False)
    for e, p in zip(engines, params):
        e.project_backward(*p)
    torch.cuda.synchronize()
    out = {"rgb": np.zeros((C, H, W, 3), np.float32), "alpha": np.zeros((C, H, W), np.float32),
           "T": np.zeros((C, H, W), np.float32), "last_gid": np.full((C, H, W), -1, np.int64)}
    for r, e in enumerate(engines):
        if e.C_loc == 0:
            continue
        out["rgb"][e.c0:e.c1] = e.out_rgb[:e.C_loc].cpu().numpy()
        out["alpha"][e.c0:e.c1] = e.out_alpha[:e.C_loc].cpu().numpy()
        out["T"][e.c0:e.c1] = e.out_T[:e.C_loc].cpu().numpy()
        # last composited splat -> its global Gaussian id (received rows are source
        # rank-major; the source's gaussian_ids are shard-local)
        item_gid = np.zeros(e.n_recv, np.int64)
        pos = 0
        for s in range(R):
            n = e.recv_splits[s]
            if n:
                o = int(np.sum(engines[s].send_splits[:r]))
                item_gid[pos:pos + n] = engines[s].gaussian_ids[o:o + n].cpu().numpy() + shard_range(N, R, s)[0]
            pos += n
        ids = e.isect_ids[:int(e.M.item())].cpu().numpy()
        offsets = e.tile_offsets.cpu().numpy()
        TX, TY = e.TX, e.TY
        ys, xs = np.mgrid[0:H, 0:W]
        tile = (ys // 16) * TX + (xs // 16)
        for c in range(e.C_loc):
            start = offsets[c * TX * TY + tile]
            li = e.last_ids[c].cpu().numpy()
            has = li >= start
            lg = out["last_gid"][e.c0 + c]
            lg[has] = (e.c0 + c) * N + item_gid[ids[li[has]]]   # flat id c*N+n
    for k in GRAD_KEYS:
        out[k] = np.concatenate([getattr(e, k).cpu().numpy() for e in engines])
    out["engines"] = engines
    return out


CASES = [("tiny_sh3_ragged", 2), ("mip_small", 3), ("mip_small_aa", 4), ("rgb_direct", 2), ("few_views", 3)]


def _case(name):
    if name == "tiny_sh3_ragged":
        return S.tiny_scene(1, N=1500, width=200, height=150, sh_degree=3, views=2), 0
    if name == "mip_small":
        return S.mipnerf_like_scene(20000, width=320, height=200, views=4, sh_degree=3, seed=11), 0
    if name == "mip_small_aa":
        return S.mipnerf_like_scene(20000, width=320, height=200, views=4, sh_degree=3, seed=12), 1
    if name == "rgb_direct":
        return S.tiny_scene(2, N=400, width=97, height=61, sh_degree=-1, views=3), 0
    if name == "few_views":   # more ranks than views: one rank renders nothing
        return S.tiny_scene(3, N=900, width=130, height=90, sh_degree=1, views=2), 0
    raise KeyError(name)


@pytest.mark.parametrize("name,R", CASES)
def test_sharded_equals_one_gpu_and_oracle(name, R):
    sc, aa = _case(name)
    C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
    v_img, _ = S.image_grads(7, C, H, W, l1_scale=False)
    o = oracle.Options(sh_degree=sc["sh_degree"], antialiased=aa)
    one = U.run_gpu(sc, antialiased=aa, v_img=v_img)
    sh = run_sharded(sc, R, v_img, antialiased=aa)
    for k in ("rgb", "alpha", "T"):
        assert np.array_equal(sh[k], one[k]), f"sharded {k} must be bit-identical to the one-GPU call"
    assert np.array_equal(sh["last_gid"], U.last_gid(one, N)), "last composited splat per pixel"
    # and the parity contract against the oracle (every pixel, every gradient element)
    ref = U.oracle_reference(sc, o, one, v_img, with_isect=False)
    U.assert_images(one, ref, label=f"shard/{name}")
    U.assert_grads(sc, sh, ref, label=f"shard/{name}", vs=one["v_splats"])
    # same kernels, fp32 atomic order only: within the atomic-order bound of the one-GPU run
    U.assert_same_kernel_grads(sc, o, ref["bwd"], sh, one, label=f"shard-vs-one/{name}")


def test_sharded_capacity_growth():
    """Too-small item / intersection capacities: the owner's nnz overflow and the renderer's
    M overflow are detected and the step re-run to the same images."""
    sc, _ = _case("tiny_sh3_ragged")
    C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
    v_img, _ = S.image_grads(8, C, H, W, l1_scale=False)
    a = run_sharded(sc, 2, v_img)
    b = run_sharded(sc, 2, v_img, nnz_capacity=5)
    assert np.array_equal(a["rgb"], b["rgb"]) and np.array_equal(a["T"], b["T"])
    o = oracle.Options(sh_degree=sc["sh_degree"])
    ob = oracle.render_bwd(oracle.project(sc, o), C, N, W, H, o, v_img.astype(np.float64))
    U.assert_same_kernel_grads(sc, o, ob, a, b, label="shard-regrow")


@pytest.mark.slow
def test_sharded_large_scene_full_scale():
    """BASELINE configs[3]'s scene (6M Gaussians, SH3, 1920x1080) sharded over R = 8 simulated
    ranks, one view each: every pixel of every view bit-identical to the one-GPU call over the
    same 8 views, the last composited splat identical, and the sharded gradients (each rank's
    750k Gaussians) equal to the one-GPU gradients up to fp32 atomic order."""
    sc = S.scene_from_config("large6m", views=8)
    C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
    v_img, _ = S.image_grads(11, C, H, W, l1_scale=False)
    # the loss restricted to 8 seeded tiles per view, so the oracle can bound the atomic order
    mask = S.tile_subset_mask(11, C, W, H, 8)
    v_img *= np.repeat(np.repeat(mask, 16, 1), 16, 2)[:, :H, :W, None]
    one = U.run_gpu(sc, v_img=v_img)
    sh = run_sharded(sc, 8, v_img)
    for k in ("rgb", "alpha", "T"):
        assert np.array_equal(sh[k], one[k]), k
    assert np.array_equal(sh["last_gid"], U.last_gid(one, N))
    o = oracle.Options(sh_degree=sc["sh_degree"])
    b = oracle.render_bwd(oracle.project(sc, o), C, N, W, H, o, v_img.astype(np.float64), tile_mask=mask)
    U.assert_same_kernel_grads(sc, o, b, sh, one, label="shard-large")
