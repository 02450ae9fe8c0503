"""GPU parity: the CUDA path (through the C-ABI) against the oracle on the same seeded
inputs.  Bit-exact for radii, projected means / depths (key path), tile keys, sorted
order and tile ranges; 1e-4 absolute on images and transmittance; 1e-3 relative (+ the
fp32 condition floor) on gradients.  See DESIGN.md "Parity contract"."""
import numpy as np
import pytest

import oracle
from synth import scenes as S
from tests import parity_util as U

pytestmark = pytest.mark.gpu


def _scene(name):
    if name == "tiny":                       # BASELINE configs[0]
        return S.tiny_scene(0), {}
    if name == "tiny_sh3_ragged":
        sc = S.tiny_scene(1, N=1500, width=200, height=150, sh_degree=3, views=2)
        return sc, {}
    if name == "mip_small":
        return S.mipnerf_like_scene(20000, width=320, height=200, views=2, sh_degree=3, seed=11), {}
    if name == "mip_small_aa":
        return S.mipnerf_like_scene(20000, width=320, height=200, views=2, sh_degree=3, seed=12), {"antialiased": 1}
    if name == "rgb_direct":
        return S.tiny_scene(2, N=400, width=97, height=61, sh_degree=-1, views=3), {}
    if name == "fig1":
        return S.fig1_scene(), {}
    raise KeyError(name)


SCENES = ["tiny", "tiny_sh3_ragged", "mip_small", "mip_small_aa", "rgb_direct", "fig1"]


def _run_both(name, with_alpha=False, bg=False, seed=0):
    """Both paths on the same inputs, the full loss (no pixel masked).  Pixels where the
    oracle meets a threshold decision within the fp32 error bound (Q28b) admit
    every outcome of those decisions; the oracle enumerates them and is compared in the
    outcome the GPU's pixel equals (U.oracle_reference)."""
    sc, kw = _scene(name)
    C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
    v_img, v_a = S.image_grads(seed, C, H, W, l1_scale=False, with_alpha=with_alpha)
    bgs = np.random.default_rng(seed).uniform(0, 1, (C, 3)).astype(np.float32) if bg else None
    aa = kw.get("antialiased", 0)
    o = oracle.Options(sh_degree=sc["sh_degree"], antialiased=aa)
    gpu = U.run_gpu(sc, antialiased=aa, v_img=v_img, v_alpha=v_a, backgrounds=bgs)
    ref = U.oracle_reference(sc, o, gpu, v_img, v_a, bgs)
    return sc, gpu, ref


@pytest.fixture(scope="module")
def cache():
    return {}


def _get(cache, name, **kw):
    key = (name, tuple(sorted(kw.items())))
    if key not in cache:
        cache[key] = _run_both(name, **kw)
    return cache[key]


@pytest.mark.parametrize("name", SCENES)
def test_project_parity(cache, name):
    sc, gpu, ref = _get(cache, name)
    p = ref["proj"]
    assert np.array_equal(gpu["radii"], p["radii"]), "radii (key path) must be bit-exact"
    vis = p["radii"][..., 0] > 0
    assert vis.any()
    sp = gpu["splats"]
    assert np.array_equal(sp[..., 0:2][vis], p["mean2d_f"][vis]), "mean2d (key path) must be bit-exact"
    assert np.array_equal(sp[..., 3][vis], p["depth_f"][vis]), "depth (key path) must be bit-exact"
    assert np.all(sp[~vis] == 0)
    np.testing.assert_allclose(sp[..., 4:7][vis], p["conic"][vis], rtol=1e-3, atol=1e-7)
    np.testing.assert_allclose(sp[..., 8:11][vis], p["rgb"][vis], rtol=1e-5, atol=1e-5)
    # slots 7, 11: blurred variances a, c = diag((Sigma'+sI)) = diag(conic^-1)
    A, B, Cc = p["conic"][..., 0][vis], p["conic"][..., 1][vis], p["conic"][..., 2][vis]
    det = A * Cc - B * B
    np.testing.assert_allclose(sp[..., 7][vis], Cc / det, rtol=1e-3)
    np.testing.assert_allclose(sp[..., 11][vis], A / det, rtol=1e-3)
    np.testing.assert_allclose(sp[..., 2][vis], p["opac_eff"][vis], rtol=1e-3, atol=1e-4)


@pytest.mark.parametrize("name", SCENES)
def test_isect_parity(cache, name):
    sc, gpu, ref = _get(cache, name)
    assert gpu["M"] == len(ref["keys"])
    assert np.array_equal(gpu["keys"], ref["keys"]), "tile keys must be bit-exact"
    assert np.array_equal(gpu["ids"], ref["ids"]), "sorted order must be bit-exact"
    assert np.array_equal(gpu["offsets"], ref["offsets"]), "tile ranges must be bit-exact"


@pytest.mark.parametrize("C,N,W,H,rmax,seed", [(3, 5000, 333, 177, 40, 5),     # ragged, off-screen, ties
                                                (2, 3000, 64, 64, 120, 6),      # bins of ~2400: P = 4096
                                                (2, 12000, 64, 64, 120, 7)])    # bins > 4096: global path
def test_isect_stagewise_ties_and_offscreen(C, N, W, H, rmax, seed):
    """Stage-wise: identical synthetic (radii, mean2d, depth) fed to both isect
    implementations, with many equal depths (tie-break by flat id, Q16), off-screen
    rectangles, zero radii, several cameras, and per-tile lists from a few entries to
    more than the shared-memory depth sort holds (K5b)."""
    import torch
    from paper_2409_06765_b200 import _lib as L
    rng = np.random.default_rng(seed)
    radii = rng.integers(1, rmax, size=(C, N, 2)).astype(np.int32)
    radii[rng.uniform(size=(C, N)) < 0.2] = 0
    m2 = np.stack([rng.uniform(-60, W + 60, (C, N)), rng.uniform(-60, H + 60, (C, N))], -1).astype(np.float32)
    depth = rng.choice(np.float32([0.5, 1.0, 1.5, 2.25, 7.0]), size=(C, N)).astype(np.float32)
    depth[radii[..., 0] == 0] = 0
    m2[radii[..., 0] == 0] = 0
    o = oracle.Options()
    proj = dict(radii=radii, mean2d_f=m2, depth_f=depth)
    keys, ids, offs = oracle.isect(proj, C, N, W, H, o)
    if rmax > 100:
        assert np.diff(offs).max() > (4096 if N > 5000 else 1024)
    dev = "cuda"
    splats = np.zeros((C, N, 12), np.float32)
    splats[..., 0:2] = m2
    splats[..., 3] = depth
    t_r = torch.from_numpy(radii).to(dev)
    t_s = torch.from_numpy(splats).to(dev)
    TX, TY = L.tiles(W, H)
    cap = len(keys) + 100
    Md = torch.zeros(1, dtype=torch.int64, device=dev)
    ov = torch.zeros(1, dtype=torch.int32, device=dev)
    gid = torch.zeros(cap, dtype=torch.int32, device=dev)
    gk = torch.zeros(cap, dtype=torch.int64, device=dev)
    go = torch.zeros(C * TX * TY + 1, dtype=torch.int32, device=dev)
    wsz = L.gs_isect_workspace_size(C, N, W, H, cap)
    ws = torch.zeros(wsz + 256, dtype=torch.uint8, device=dev)
    a = (-ws.data_ptr()) % 256
    L.gs_isect_tiles(L.options(), C, N, W, H, t_r, t_s, cap, Md, ov, gid, gk, go, ws[a:a + wsz])
    torch.cuda.synchronize()
    M = int(Md.item())
    assert M == len(keys) and int(ov.item()) == 0
    assert np.array_equal(gk[:M].cpu().numpy().view(np.uint64), keys)
    assert np.array_equal(gid[:M].cpu().numpy(), ids)
    assert np.array_equal(go.cpu().numpy(), offs)
    # overflow path: capacity below M sets the flag and reports the true M
    cap2 = M // 2
    wsz2 = L.gs_isect_workspace_size(C, N, W, H, cap2)
    ws2 = torch.zeros(wsz2 + 256, dtype=torch.uint8, device=dev)
    a2 = (-ws2.data_ptr()) % 256
    L.gs_isect_tiles(L.options(), C, N, W, H, t_r, t_s, cap2, Md, ov, gid, None, go, ws2[a2:a2 + wsz2])
    torch.cuda.synchronize()
    assert int(Md.item()) == M and int(ov.item()) == 1


@pytest.mark.parametrize("name", SCENES)
def test_raster_fwd_parity(cache, name):
    """Every pixel: colour, T, alpha within 1e-4 and the same last composited splat; the
    ambiguous ones (reported) against the oracle's outcome the GPU took."""
    sc, gpu, ref = _get(cache, name)
    U.assert_images(gpu, ref, label=name)
    a = ref["amb"]
    print(name, U.amb_report(ref))
    assert a["ambiguous"] <= 1e-3 * a["pixels"] + 1, U.amb_report(ref)


@pytest.mark.parametrize("name", SCENES)
def test_backward_parity(cache, name):
    """Every 2D record-gradient element and every parameter-gradient element."""
    sc, gpu, ref = _get(cache, name)
    U.assert_grads(sc, gpu, ref, label=f"backward/{name}")


def test_background_and_alpha_gradient(cache):
    sc, gpu, ref = _get(cache, "tiny_sh3_ragged", with_alpha=True, bg=True)
    U.assert_images(gpu, ref, label="bg+alpha")
    U.assert_grads(sc, gpu, ref, label="bg+alpha")


def test_edge_cases():
    # empty scene
    sc = S.tiny_scene(0, N=1)
    sc = {k: (v[:0] if isinstance(v, np.ndarray) and k in ("means", "quats", "scales", "opacities", "colors") else v)
          for k, v in sc.items()}
    gpu = U.run_gpu(sc)
    assert gpu["M"] == 0 and np.all(gpu["rgb"] == 0) and np.all(gpu["T"] == 1)
    # everything behind the camera
    sc = S.tiny_scene(3, N=50)
    sc["means"][:, 2] = -1.0
    gpu = U.run_gpu(sc)
    assert gpu["M"] == 0 and np.all(gpu["radii"] == 0) and np.all(gpu["v_means"] == 0)
    # zero quaternion and zero opacity
    sc = S.tiny_scene(4, N=50)
    sc["quats"][:10] = 0
    sc["opacities"][10:20] = 0
    ref = oracle.project(sc, oracle.Options(sh_degree=0))
    gpu = U.run_gpu(sc)
    assert np.array_equal(gpu["radii"], ref["radii"])
    assert np.all(gpu["radii"][:, :10] == 0)
    assert np.all(np.isfinite(gpu["v_quats"])) and np.all(gpu["v_quats"][:10] == 0)


def test_determinism():
    sc = S.mipnerf_like_scene(20000, width=320, height=200, views=2, sh_degree=3, seed=21)
    v, _ = S.image_grads(0, 2, 200, 320, l1_scale=False)
    a = U.run_gpu(sc, v_img=v)
    b = U.run_gpu(sc, v_img=v)
    for k in ["radii", "splats", "keys", "ids", "offsets", "rgb", "T", "last_ids"]:
        assert np.array_equal(a[k], b[k]), k


def test_rasterization_api_autograd():
    import torch
    from paper_2409_06765_b200 import rasterization
    sc = S.tiny_scene(1, N=1500, width=200, height=150, sh_degree=3, views=2)
    dev = "cuda"
    ts = [t.clone().requires_grad_(i < 5) for i, t in enumerate(U.to_torch(sc, dev))]
    rgb, alpha, meta = rasterization(*ts, 200, 150, sh_degree=3)
    v, va = S.image_grads(3, 2, 150, 200, l1_scale=False, with_alpha=True)
    loss = (rgb * torch.from_numpy(v).to(dev)).sum() + (alpha[..., 0] * torch.from_numpy(va).to(dev)).sum()
    loss.backward()
    gpu = U.run_gpu(sc, v_img=v, v_alpha=va)
    assert np.array_equal(rgb.detach().cpu().numpy(), gpu["rgb"])
    # same kernels, different fp32 atomic order only
    o = oracle.Options(sh_degree=3)
    b = oracle.render_bwd(oracle.project(sc, o), 2, 1500, 200, 150, o, v.astype(np.float64), va.astype(np.float64))
    api = {k: t.grad.cpu().numpy() for t, k in zip(ts[:5], U.GRAD_KEYS)}
    U.assert_same_kernel_grads(sc, o, b, api, gpu, label="api")
    assert meta["means2d"].shape == (2, 1500, 2) and meta["radii"].dtype == torch.int32
    # packed mode through the same API: bit-identical images (Q29), same gradients up to atomic order
    tp = [t.detach().clone().requires_grad_(i < 5) for i, t in enumerate(ts)]
    rgb_p, alpha_p, meta_p = rasterization(*tp, 200, 150, sh_degree=3, packed=True)
    assert torch.equal(rgb_p, rgb) and torch.equal(alpha_p, alpha)
    nnz = meta_p["camera_ids"].numel()
    assert meta_p["means2d"].shape == (nnz, 2) and nnz == int((meta["radii"][..., 0] > 0).sum())
    loss_p = (rgb_p * torch.from_numpy(v).to(dev)).sum() + (alpha_p[..., 0] * torch.from_numpy(va).to(dev)).sum()
    loss_p.backward()
    U.assert_same_kernel_grads(sc, o, b, {k: t.grad.cpu().numpy() for t, k in zip(tp[:5], U.GRAD_KEYS)}, api,
                               label="api-packed")


def test_absgrad():
    sc = S.tiny_scene(1, N=1500, width=200, height=150, sh_degree=3, views=1)
    v, _ = S.image_grads(3, 1, 150, 200, l1_scale=False)
    gpu = U.run_gpu(sc, v_img=v, absgrad=True)
    vs = gpu["v_splats"]
    assert np.all(vs[..., 10] >= np.abs(vs[..., 0]) * (1 - 1e-5) - 1e-7)
    assert np.all(vs[..., 11] >= np.abs(vs[..., 1]) * (1 - 1e-5) - 1e-7)


def _full_scale_sampled(cfg_name, views=None, n_tiles=32, seed=0, packed=False, antialiased=False):
    """A BASELINE config at full size, in the launch configuration bench.py times (one GPU,
    all of that GPU's views in one call): key path, tile keys / order / ranges bit-exact over
    every view; images and the gradients of the loss restricted to n_tiles seeded tiles per
    view (exact for that loss, SURVEY 8c 'cheap parity for large configs'), every pixel of
    those tiles and every gradient element."""
    sc = S.scene_from_config(cfg_name, views=views)
    C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
    mask = S.tile_subset_mask(seed, C, W, H, n_tiles)
    pm = np.repeat(np.repeat(mask, 16, 1), 16, 2)[:, :H, :W]
    v_img, _ = S.image_grads(seed, C, H, W, l1_scale=False)
    v_img *= pm[..., None]
    o = oracle.Options(sh_degree=sc["sh_degree"], antialiased=int(antialiased))
    gpu = U.run_gpu(sc, antialiased=antialiased, v_img=v_img, packed=packed)
    ref = U.oracle_reference(sc, o, gpu, v_img, tile_mask=mask)
    p = ref["proj"]
    vis = (p["radii"][..., 0] > 0) & (p["radii"][..., 1] > 0)
    keys, ids, offs = ref["keys"], ref["ids"], ref["offsets"]
    if packed:
        cam, gid, index = oracle.pack(p)
        assert np.array_equal(gpu["camera_ids"], cam) and np.array_equal(gpu["gaussian_ids"], gid)
        assert np.array_equal(gpu["radii"], p["radii"][cam, gid])
        assert np.array_equal(gpu["splats"][:, 0:2], p["mean2d_f"][cam, gid])
        assert np.array_equal(gpu["splats"][:, 3], p["depth_f"][cam, gid])
        assert np.array_equal(gpu["ids"], index.reshape(-1)[ids])
    else:
        assert np.array_equal(gpu["radii"], p["radii"])
        assert np.array_equal(gpu["splats"][..., 0:2][vis], p["mean2d_f"][vis])
        assert np.array_equal(gpu["splats"][..., 3][vis], p["depth_f"][vis])
        assert np.array_equal(gpu["ids"], ids)
    assert np.array_equal(gpu["keys"], keys)
    assert np.array_equal(gpu["offsets"], offs)
    U.assert_images(gpu, ref, sel=pm.astype(bool), label=cfg_name)
    print(cfg_name, U.amb_report(ref))
    U.assert_grads(sc, gpu, ref, label=cfg_name, packed=packed)
    return len(keys)


@pytest.mark.slow
def test_config2_full_scale_sampled():
    """BASELINE configs[1]: 1M Gaussians, SH3, one 1297x840 view (the bench workload)."""
    _full_scale_sampled("garden1m")


@pytest.mark.slow
def test_config3_batch_full_scale_sampled():
    """BASELINE configs[2]: 3M Gaussians, 8 views of 1297x840 in one call (the N=1 shard of
    the 1/2/4/8-GPU view-parallel run)."""
    _full_scale_sampled("batch3m", n_tiles=16, seed=3)


@pytest.mark.slow
def test_config4_large_shard_full_scale_sampled():
    """BASELINE configs[3]: 6M Gaussians, SH3, 1920x1080 -- one GPU's shard of the 32-view,
    8-GPU step (4 views in one call)."""
    _full_scale_sampled("large6m", views=4, n_tiles=16, seed=4)


# ---- packed mode (Q29, BASELINE configs[4]) -------------------------------------------
@pytest.mark.parametrize("name", ["tiny_sh3_ragged", "mip_small_aa", "rgb_direct"])
def test_packed_parity(name):
    """Packed items = the oracle's pack() of the visible set; records bit-identical to the
    dense path's rows; keys bit-exact with packed values; images bit-identical to the dense
    path (Q29); gradients against the oracle."""
    sc, kw = _scene(name)
    aa = kw.get("antialiased", 0)
    C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
    v_img, _ = S.image_grads(4, C, H, W, l1_scale=False)
    o = oracle.Options(sh_degree=sc["sh_degree"], antialiased=aa)
    dense = U.run_gpu(sc, antialiased=aa, v_img=v_img)
    pk = U.run_gpu(sc, antialiased=aa, v_img=v_img, packed=True)
    ref = U.oracle_reference(sc, o, pk, v_img, with_isect=False)
    p = ref["proj"]
    cam, gid, index = oracle.pack(p)
    assert pk["nnz"] == cam.size
    assert np.array_equal(pk["camera_ids"], cam) and np.array_equal(pk["gaussian_ids"], gid)
    assert np.array_equal(pk["radii"], dense["radii"][cam, gid])
    assert np.array_equal(pk["splats"], dense["splats"][cam, gid])
    keys, ids, offs = oracle.isect(p, C, N, W, H, o)
    assert np.array_equal(pk["keys"], keys), "tile keys must be bit-exact"
    assert np.array_equal(pk["ids"], index.reshape(-1)[ids]), "sorted order (packed values) must be bit-exact"
    assert np.array_equal(pk["offsets"], offs)
    for k in ("rgb", "alpha", "T", "last_ids"):
        assert np.array_equal(pk[k], dense[k]), f"packed {k} must be bit-identical to dense (Q29)"
    U.assert_images(pk, ref, label=f"packed/{name}")
    U.assert_grads(sc, pk, ref, label=f"packed/{name}", packed=True)


def test_packed_capacity_growth():
    """A too-small nnz capacity sets the device overflow flag; run_checked grows it and
    re-runs to the same result."""
    sc, _ = _scene("tiny_sh3_ragged")
    a = U.run_gpu(sc, packed=True)
    b = U.run_gpu(sc, packed=True, nnz_capacity=7, cap=16)
    assert a["nnz"] == b["nnz"] > 7
    assert np.array_equal(a["rgb"], b["rgb"]) and np.array_equal(a["ids"], b["ids"])


@pytest.mark.slow
def test_config5_aa_packed_full_scale_sampled():
    """BASELINE configs[4]: 1M Gaussians, antialiased, packed, 4 views of 1297x840."""
    _full_scale_sampled("aa_packed1m", seed=5, packed=True, antialiased=True)


# ---- depth rendering (NEXT-2) and camera pose gradients (NEXT-3) ----
DEPTH_RTOL = 1e-5        # depth maps: fp32 sums of z alpha T, relative to the scene depth scale


@pytest.mark.parametrize("name,mode,packed", [("tiny_sh3_ragged", 1, False), ("mip_small", 2, False),
                                              ("mip_small_aa", 2, True), ("rgb_direct", 1, False)])
def test_depth_and_pose_parity(name, mode, packed):
    """Depth channel (accumulated, mode 1; expected, mode 2) against the oracle; its gradients
    into v_splats slot 3 and through t_z; camera pose gradients against the oracle's."""
    sc, kw = _scene(name)
    aa = kw.get("antialiased", 0)
    C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
    v_img, _ = S.image_grads(7, C, H, W, l1_scale=False)
    v_d = np.random.default_rng(8).normal(size=(C, H, W)).astype(np.float32) * 0.05
    o = oracle.Options(sh_degree=sc["sh_degree"], antialiased=aa)
    gpu = U.run_gpu(sc, antialiased=aa, v_img=v_img, depth_mode=mode, v_depth=v_d, pose=True, packed=packed)
    ref = U.oracle_reference(sc, o, gpu, v_img, depth_mode=mode, v_depth=v_d, pose=True, with_isect=False)
    f, p = ref["fwd"], ref["proj"]
    ref_d = f["depth"] if mode == 1 else f["depth_exp"]
    zmax = np.abs(p["depth"][p["radii"][..., 0] > 0]).max()
    assert np.abs(gpu["depth"] - ref_d).max() <= DEPTH_RTOL * zmax + U.IMG_ATOL
    U.assert_images(gpu, ref, label=f"depth/{name}")
    # slot 3 (d L / d depth of each (c, n)) with the same model as the 2D slots; pose per entry
    U.assert_grads(sc, gpu, ref, label=f"depth+pose/{name}", packed=packed, pose=True, depth=True)


def test_render_modes_api():
    """render_mode through the public API: RGB+ED = [RGB | expected depth] and its gradients
    equal the engine's; viewmats.requires_grad yields the pose gradient."""
    import torch
    from paper_2409_06765_b200 import rasterization
    sc = S.tiny_scene(1, N=1500, width=200, height=150, sh_degree=3, views=2)
    dev = "cuda"
    ts = [t.clone().requires_grad_(i < 6) for i, t in enumerate(U.to_torch(sc, dev))]
    out, alpha, meta = rasterization(*ts, 200, 150, sh_degree=3, render_mode="RGB+ED")
    assert out.shape == (2, 150, 200, 4)
    v, _ = S.image_grads(3, 2, 150, 200, l1_scale=False)
    vd = np.random.default_rng(9).normal(size=(2, 150, 200)).astype(np.float32) * 0.05
    loss = (out[..., :3] * torch.from_numpy(v).to(dev)).sum() + (out[..., 3] * torch.from_numpy(vd).to(dev)).sum()
    loss.backward()
    gpu = U.run_gpu(sc, v_img=v, depth_mode=2, v_depth=vd, pose=True)
    assert np.array_equal(out[..., 3].detach().cpu().numpy(), gpu["depth"])
    o = oracle.Options(sh_degree=3)
    b = oracle.render_bwd(oracle.project(sc, o), 2, 1500, 200, 150, o, v.astype(np.float64),
                          v_depth_exp=vd.astype(np.float64))
    api = {k: t.grad.cpu().numpy() for t, k in zip(ts[:6], list(U.GRAD_KEYS) + ["v_viewmats"])}
    U.assert_same_kernel_grads(sc, o, b, api, gpu, label="render_modes", depth=True, pose=True)
    d, _, _ = rasterization(*[t.detach() for t in ts], 200, 150, sh_degree=3, render_mode="D")
    assert d.shape == (2, 150, 200, 1)


# ---- N-D feature rasterization (NEXT-2) ------------------------------------
@pytest.mark.parametrize("D,packed,name", [(1, False, "tiny_sh3_ragged"), (5, False, "mip_small"),
                                           (8, True, "mip_small_aa"), (13, False, "rgb_direct")])
def test_nd_features_parity(D, packed, name):
    """D-channel features through the public API (channel-chunked passes of K6/K7) against
    the oracle: feature images, the feature gradient (summed over cameras), the geometry
    gradients of the record, and the parameter gradients through the projection."""
    import torch
    from paper_2409_06765_b200 import rasterization
    sc, kw = _scene(name)
    aa = kw.get("antialiased", 0)
    C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
    rng = np.random.default_rng(D)
    feats = rng.normal(size=(N, D)).astype(np.float32)
    bg = rng.uniform(size=(C, D)).astype(np.float32)
    v_f = rng.normal(size=(C, H, W, D)).astype(np.float32)
    v_a = rng.normal(size=(C, H, W)).astype(np.float32)
    sc_o = dict(sc)
    sc_o["colors"] = np.zeros((N, 3), np.float32)
    sc_o["sh_degree"] = -1
    o = oracle.Options(sh_degree=-1, antialiased=aa)
    dev = "cuda"
    ts = [t.clone().requires_grad_(True) for t in U.to_torch(sc_o, dev)[:5]]
    ts[4] = torch.from_numpy(feats).to(dev).requires_grad_(True)
    vm, Ks = [t.clone() for t in U.to_torch(sc_o, dev)[5:]]
    out, alpha, meta = rasterization(*ts, vm, Ks, W, H, backgrounds=torch.from_numpy(bg).to(dev),
                                     rasterize_mode="antialiased" if aa else "classic", packed=packed)
    assert out.shape == (C, H, W, D)
    loss = (out * torch.from_numpy(v_f).to(dev)).sum() + (alpha[..., 0] * torch.from_numpy(v_a).to(dev)).sum()
    loss.backward()
    # the GPU run as the parity helpers see it (meta of the public API)
    gpu = dict(T=meta["T_final"].cpu().numpy(), last_ids=meta["last_ids"].cpu().numpy(),
               offsets=meta["tile_offsets"].cpu().numpy(), ids=meta["isect_ids"].cpu().numpy(),
               alpha=alpha[..., 0].detach().cpu().numpy())
    if packed:
        gpu.update(camera_ids=meta["camera_ids"].cpu().numpy(), gaussian_ids=meta["gaussian_ids"].cpu().numpy())
    img = out.detach().cpu().numpy()
    ref = U.oracle_reference(sc_o, o, gpu, v_f, v_a, bg, feats=feats, img=img, with_isect=False)
    U.assert_images(gpu, ref, img=img, key="feat", atol=U.IMG_ATOL * (1 + np.abs(ref["fwd"]["feat"]).max()),
                    label=f"nd/{D}")
    b = ref["bwd"]
    # feature gradients (summed over cameras): every element, with the floors of the rgb slots
    gf, rf = ts[4].grad.cpu().numpy().astype(np.float64), b["v_colors"]
    tol = U.GRAD_RTOL * np.abs(rf) + U.GRAD2D_FLOOR * b["a_colors"] + U.GRAD2D_ULP * b["s_colors"] + \
        b["d_colors"] + 1e-30
    assert not (np.abs(gf - rf) > tol).any(), int((np.abs(gf - rf) > tol).sum())
    vs = meta["cfg"]["v_splats"].cpu().numpy()
    if packed:
        vs = U.unpack(vs[:meta["camera_ids"].numel()], meta["camera_ids"].cpu().numpy(),
                      meta["gaussian_ids"].cpu().numpy(), C, N)
    grads = {k: t.grad.cpu().numpy() for t, k in zip(ts[:4], ["v_means", "v_quats", "v_scales", "v_opacities"])}
    U.assert_grads(sc_o, grads, ref, label=f"nd/{D}", vs=vs, keys=("v_means", "v_quats", "v_scales", "v_opacities"))


def _full_parity(sc, v_seed=0, pose=False, **kw):
    """Both paths on the same inputs with the standard contract (U.oracle_reference)."""
    C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
    v_img, _ = S.image_grads(v_seed, C, H, W, l1_scale=False)
    o = oracle.Options(sh_degree=sc["sh_degree"])
    gpu = U.run_gpu(sc, v_img=v_img, pose=pose, **kw)
    ref = U.oracle_reference(sc, o, gpu, v_img, pose=pose)
    p = ref["proj"]
    assert np.array_equal(gpu["radii"], p["radii"])
    assert np.array_equal(gpu["keys"], ref["keys"]) and np.array_equal(gpu["ids"], ref["ids"])
    U.assert_images(gpu, ref, label="full")
    U.assert_grads(sc, gpu, ref, label="full", pose=pose)
    return sc, gpu, ref["grads"], p


def _needle_scene():
    """Extremely elongated diagonal splats: ill-conditioned 2D conics (cond up to ~1e5), the
    case where the support test falls back to the axis-aligned box (DESIGN K6)."""
    sc = S.tiny_scene(11, N=300, width=160, height=120, sh_degree=1, views=1)
    rng = np.random.default_rng(11)
    k = 120
    sc["scales"][:k] = np.stack([rng.uniform(2.0, 12.0, k), np.full(k, 1e-4), np.full(k, 1e-4)], 1)
    ang = rng.uniform(0, np.pi, k)
    # rotation about the view axis z (quaternion w, x, y, z): the long axis lies diagonally
    sc["quats"][:k] = np.stack([np.cos(ang / 2), 0 * ang, 0 * ang, np.sin(ang / 2)], 1)
    sc["opacities"][:k] = 0.9
    return sc, k


@pytest.mark.parametrize("name", ["needles", "mip_small", "fig1", "tiny_sh3_ragged"])
def test_support_culling_is_output_invariant(name):
    """The conservative alpha-support test (DESIGN K6) only skips (splat, 4x4 block) pairs
    whose pixels would all skip the splat anyway: with it disabled (support_cull = 0, every
    pair of the tile evaluated) the images, T and last_ids are bit-identical and the
    gradients equal up to fp32 atomic order -- including ill-conditioned splats, which take
    the box fallback."""
    if name == "needles":
        sc, k = _needle_scene()
        p = oracle.project(sc, oracle.Options(sh_degree=1))
        A, B, Cc = p["conic"][0, :k, 0], p["conic"][0, :k, 1], p["conic"][0, :k, 2]
        vis = p["radii"][0, :k, 0] > 0
        with np.errstate(divide="ignore", invalid="ignore"):
            cond = (Cc / (A * Cc - B * B)) * A
        assert (cond[vis] > 1e4).sum() >= 5, "the scene must exercise the ill-conditioned box fallback"
    else:
        sc, _ = _scene(name)
    C, H, W = sc["viewmats"].shape[0], sc["height"], sc["width"]
    v_img, _ = S.image_grads(9, C, H, W, l1_scale=False)
    on = U.run_gpu(sc, v_img=v_img)
    off = U.run_gpu(sc, v_img=v_img, support_cull=False)
    for key in ("rgb", "alpha", "T", "last_ids", "ids", "offsets"):
        assert np.array_equal(on[key], off[key]), key
    # gradients: the same per-pixel terms summed in another fp32 atomic order -- within the
    # atomic-order bound (U.atomic_order_tol2d, from the oracle's term counts and magnitudes),
    # carried through the projection backward for the parameter gradients
    o = oracle.Options(sh_degree=sc["sh_degree"])
    p = oracle.project(sc, o)
    N = sc["means"].shape[0]
    b = oracle.render_bwd(p, C, N, W, H, o, v_img.astype(np.float64))
    U.assert_same_kernel_grads(sc, o, b, on, off, label=f"support/{name}", vs_one=on["v_splats"],
                               vs_other=off["v_splats"])


def test_many_cameras_and_pose():
    """70 views in one call (more than one 64-camera chunk of K1) with pose gradients."""
    sc = S.tiny_scene(12, N=400, width=48, height=40, sh_degree=2, views=70)
    _full_parity(sc, pose=True)


# ---- opacity-aware tile extent (bbox_mode 2, NEXT-4(ii), Q36) ---------------------------
@pytest.mark.parametrize("name,packed", [("tiny_sh3_ragged", False), ("mip_small", False), ("mip_small_aa", False),
                                         ("rgb_direct", False), ("fig1", False), ("mip_small_aa", True)])
def test_opacity_aware_extent(name, packed):
    """Radii, tile keys, sorted order and ranges bit-exact against the oracle's mode 2; fewer
    intersections than the 3-sigma box; images, T and the last composited splat per pixel
    bit-identical to mode 0 (output invariance), gradients equal up to fp32 atomic order."""
    sc, kw = _scene(name)
    aa = kw.get("antialiased", 0)
    C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
    v_img, _ = S.image_grads(9, C, H, W, l1_scale=False)
    o2 = oracle.Options(sh_degree=sc["sh_degree"], antialiased=aa, bbox_mode=2)
    p2 = oracle.project(sc, o2)
    keys, ids, offs = oracle.isect(p2, C, N, W, H, o2)
    g0 = U.run_gpu(sc, antialiased=aa, v_img=v_img, packed=packed)
    g2 = U.run_gpu(sc, antialiased=aa, v_img=v_img, packed=packed, bbox_mode=2)
    if packed:
        cam, gid, index = oracle.pack(p2)
        assert np.array_equal(g2["radii"], p2["radii"][cam, gid])
        assert np.array_equal(g2["ids"], index.reshape(-1)[ids])
    else:
        assert np.array_equal(g2["radii"], p2["radii"]), "mode-2 radii must be bit-exact"
        assert np.array_equal(g2["ids"], ids), "sorted order must be bit-exact"
    assert np.array_equal(g2["keys"], keys), "tile keys must be bit-exact"
    assert np.array_equal(g2["offsets"], offs)
    assert g2["M"] <= g0["M"]
    for k in ("rgb", "alpha", "T"):
        assert np.array_equal(g2[k], g0[k]), f"{k} must be bit-identical to the 3-sigma box"
    assert np.array_equal(U.last_gid(g2, N), U.last_gid(g0, N))
    # the same per-pixel terms in another atomic order (fewer bins, same walks)
    o0 = oracle.Options(sh_degree=sc["sh_degree"], antialiased=aa)
    b = oracle.render_bwd(oracle.project(sc, o0), C, N, W, H, o0, v_img.astype(np.float64))
    vs0, vs2 = g0["v_splats"], g2["v_splats"]
    if packed:
        vs0 = U.unpack(vs0, g0["camera_ids"], g0["gaussian_ids"], C, N)
        vs2 = U.unpack(vs2, g2["camera_ids"], g2["gaussian_ids"], C, N)
    U.assert_same_kernel_grads(sc, o0, b, g2, g0, label=f"bbox2/{name}", vs_one=vs2, vs_other=vs0)


# ---- NEXT-1: Absgrad parity and densification statistics (App. ADC / Absgrad P:196-206) ---
@pytest.mark.parametrize("name,packed", [("tiny_sh3_ragged", False), ("mip_small", False), ("mip_small_aa", True)])
def test_absgrad_parity_and_densify_stats(name, packed):
    import torch
    from paper_2409_06765_b200 import _lib as L
    sc, kw = _scene(name)
    aa = kw.get("antialiased", 0)
    C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
    v_img, _ = S.image_grads(12, C, H, W, l1_scale=False)
    o = oracle.Options(sh_degree=sc["sh_degree"], antialiased=aa)
    gpu = U.run_gpu(sc, antialiased=aa, v_img=v_img, absgrad=True, packed=packed)
    ref = U.oracle_reference(sc, o, gpu, v_img, with_isect=False)
    p, b = ref["proj"], ref["bwd"]
    vis = (p["radii"][..., 0] > 0)
    if packed:
        cam, gid, _ = oracle.pack(p)
        vs = U.unpack(gpu["v_splats"], cam, gid, C, N)
        radii_dense = U.unpack(gpu["radii"], cam, gid, C, N)
    else:
        vs, radii_dense = gpu["v_splats"], gpu["radii"]
    ag = np.stack([vs[..., 10], vs[..., 11]], axis=-1)
    bad = U.check_grad2d(ag, b["absgrad"], b["a2d"][..., 0:2], vis, b["s2d"][..., 0:2], b["d2d"][..., 0:2])
    assert bad.sum() == 0, bad.sum()
    # statistics from the GPU's own radii / v_splats (inputs), both flavours, accumulated twice
    eng = gpu["engine"]
    dev = "cuda"
    for absgrad in (False, True):
        g2 = torch.zeros(N, device=dev)
        cnt = torch.zeros(N, dtype=torch.int32, device=dev)
        mr = torch.zeros(N, device=dev)
        for _ in range(2):
            if packed:
                L.gs_densify_stats(eng.opts, N, C, eng.radii, eng.v_splats, g2, cnt, mr, absgrad=absgrad,
                                   scale=(W / 2, H / 2), radius_scale=1 / max(W, H), nnz_capacity=eng.nnz_cap,
                                   nnz=eng.nnz, gaussian_ids=eng.gaussian_ids)
            else:
                L.gs_densify_stats(eng.opts, N, C, eng.radii, eng.v_splats, g2, cnt, mr, absgrad=absgrad,
                                   scale=(W / 2, H / 2), radius_scale=1 / max(W, H))
        torch.cuda.synchronize()
        g_in = ag if absgrad else vs[..., 0:2]
        ref = oracle.densify_stats(radii_dense, g_in, scale=(W / 2, H / 2), radius_scale=1 / max(W, H))
        np.testing.assert_allclose(g2.cpu().numpy(), 2 * ref["grad2d"], rtol=1e-5, atol=1e-30)
        assert np.array_equal(cnt.cpu().numpy(), 2 * ref["count"])
        np.testing.assert_allclose(mr.cpu().numpy(), ref["max_radii"], rtol=1e-6)


def test_cuda_graph_replay_equals_eager():
    """Engine.capture(): one step recorded into a CUDA graph replays to the eager step's
    images bit for bit and its gradients up to fp32 atomic order."""
    import torch
    sc = S.mipnerf_like_scene(20000, width=320, height=200, views=2, sh_degree=3, seed=11)
    C, N, W, H = 2, 20000, 320, 200
    v_img, _ = S.image_grads(0, C, H, W, l1_scale=False)
    eager = U.run_gpu(sc, v_img=v_img)
    eng = eager["engine"]
    params = U.to_torch(sc, "cuda")
    v = torch.from_numpy(v_img).cuda()
    eng.run_checked(params, v)
    eng.capture(params, v)
    for t in (eng.out_rgb, eng.flat_grad):
        t.zero_()
    eng.replay()
    eng.replay()
    torch.cuda.synchronize()
    assert int(eng.overflow.item()) == 0
    assert np.array_equal(eng.out_rgb.cpu().numpy(), eager["rgb"])
    assert np.array_equal(eng.out_T.cpu().numpy(), eager["T"])
    o = oracle.Options(sh_degree=3)
    b = oracle.render_bwd(oracle.project(sc, o), C, N, W, H, o, v_img.astype(np.float64))
    rep = {k: getattr(eng, k).cpu().numpy() for k in U.GRAD_KEYS}
    U.assert_same_kernel_grads(sc, o, b, rep, eager, label="graph", vs_one=eng.v_splats.cpu().numpy(),
                               vs_other=eager["v_splats"])


def test_project_bwd_range_equals_whole():
    """gs_project_bwd_range over buckets (the data-parallel gradient buckets) writes exactly the
    rows gs_project_bwd writes, bit for bit, from the same record gradients."""
    import torch
    from paper_2409_06765_b200 import _lib as L
    from paper_2409_06765_b200 import dist as D
    sc = S.mipnerf_like_scene(20000, width=320, height=200, views=2, sh_degree=3, seed=11)
    v_img, _ = S.image_grads(0, 2, 200, 320, l1_scale=False)
    gpu = U.run_gpu(sc, v_img=v_img)
    eng = gpu["engine"]
    p = U.to_torch(sc, "cuda")
    lay, total = D.bucket_layout(20000, 16, True, n_buckets=3)
    flat = torch.full((total,), float("nan"), device="cuda")
    for b in D.bucket_views(flat, lay):
        L.gs_project_bwd_range(eng.opts, b["n0"], b["n1"], *p[:5], 16, p[5], p[6], 320, 200, eng.radii, eng.v_splats,
                               b["means"], b["quats"], b["scales"], b["opacities"], b["colors"])
    torch.cuda.synchronize()
    g = D.gather_buckets(flat, lay)
    for k in ("means", "quats", "scales", "opacities", "colors"):
        assert torch.equal(g[k], getattr(eng, "v_" + k)), k


@pytest.mark.parametrize("name", ["tiny_sh3_ragged", "mip_small", "rgb_direct"])
def test_bbox_mode1_square_box(name):
    """bbox_mode 1 (Q12 option: the square 3 sqrt(lambda_max) box of 3DGS): radii, tile keys,
    sorted order and ranges bit-exact against the oracle's mode 1, and the full image /
    gradient contract against it (its support predicate is the square box)."""
    sc, kw = _scene(name)
    aa = kw.get("antialiased", 0)
    C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
    v_img, _ = S.image_grads(13, C, H, W, l1_scale=False)
    o = oracle.Options(sh_degree=sc["sh_degree"], antialiased=aa, bbox_mode=1)
    gpu = U.run_gpu(sc, antialiased=aa, v_img=v_img, bbox_mode=1)
    ref = U.oracle_reference(sc, o, gpu, v_img)
    p = ref["proj"]
    assert np.array_equal(gpu["radii"], p["radii"])
    vis = p["radii"][..., 0] > 0
    assert np.all(p["radii"][..., 0][vis] == p["radii"][..., 1][vis])      # square
    assert np.array_equal(gpu["keys"], ref["keys"]) and np.array_equal(gpu["ids"], ref["ids"])
    assert np.array_equal(gpu["offsets"], ref["offsets"])
    U.assert_images(gpu, ref, label=f"bbox1/{name}")
    U.assert_grads(sc, gpu, ref, label=f"bbox1/{name}")


def test_tile_order_is_a_permutation_and_output_invariant():
    """gs_tile_order: a permutation of the bins, camera by camera, each camera's tiles in
    non-increasing length bucket; gs_rasterize_bwd launched in that order, with the record
    gradients zero-filled on the side stream (bwd_zero_fill = 0), gives the natural order's
    in-call zero-fill gradients up to fp32 atomic order (same-kernel bound)."""
    import torch
    sc = S.mipnerf_like_scene(20000, width=320, height=200, views=2, sh_degree=3, seed=11)
    C, N, W, H = 2, 20000, 320, 200
    v_img, _ = S.image_grads(0, C, H, W, l1_scale=False)
    ordered = U.run_gpu(sc, v_img=v_img)             # Engine default: tile order + side-stream prep on
    natural = U.run_gpu(sc, v_img=v_img, tile_order=False, overlap_prep=False)
    eng = ordered["engine"]
    TT = eng.TX * eng.TY
    order = eng.tile_order.cpu().numpy()
    offs = ordered["offsets"]
    assert np.array_equal(np.sort(order), np.arange(C * TT))
    for c in range(C):
        oc = order[c * TT:(c + 1) * TT]
        assert np.all((oc >= c * TT) & (oc < (c + 1) * TT))
        bucket = np.minimum(255, (offs[oc + 1] - offs[oc]) >> 4)
        assert np.all(np.diff(bucket) <= 0)
    for k in ["rgb", "T", "last_ids"]:
        assert np.array_equal(ordered[k], natural[k]), k
    o = oracle.Options(sh_degree=3)
    b = oracle.render_bwd(oracle.project(sc, o), C, N, W, H, o, v_img.astype(np.float64))
    rep = {k: natural[k] for k in U.GRAD_KEYS}
    U.assert_same_kernel_grads(sc, o, b, rep, ordered, label="tile-order", vs_one=natural["v_splats"],
                               vs_other=ordered["v_splats"])


# seeded sweep: shapes, SH degrees 0-3 (1 and 2 appear nowhere else), classic / antialiased,
# backgrounds and the alpha-output gradient, both scene generators -- every stage's full
# contract (bit-exact keys, order, ranges, radii, mu', depth; images; every gradient element)
def _sweep_cases():
    rng = np.random.default_rng(2409)
    cases = []
    for i in range(32):
        mip = i % 3 == 2
        sh = int(rng.integers(0, 4))
        small = i % 8 == 7   # images of one or two partial tiles
        cases.append(dict(seed=100 + i, mip=mip, N=int(rng.integers(3000, 12000)) if mip else int(rng.integers(50, 2500)),
                          W=int(rng.integers(5, 33)) if small else int(rng.integers(40, 260)),
                          H=int(rng.integers(5, 33)) if small else int(rng.integers(30, 200)),
                          views=int(rng.integers(1, 6)),
                          sh=sh if i != 0 else 1, aa=int(rng.integers(0, 2)), bg=bool(rng.integers(0, 2))))
    cases[1]["sh"] = 2
    return cases


@pytest.mark.parametrize("case", _sweep_cases(), ids=lambda c: f"s{c['seed']}")
def test_seeded_sweep_full_contract(case):
    c = case
    if c["mip"]:
        sc = S.mipnerf_like_scene(c["N"], width=c["W"], height=c["H"], views=c["views"], sh_degree=c["sh"],
                                  seed=c["seed"])
    else:
        sc = S.tiny_scene(c["seed"], N=c["N"], width=c["W"], height=c["H"], sh_degree=c["sh"], views=c["views"])
    C, W, H = sc["viewmats"].shape[0], sc["width"], sc["height"]
    v_img, v_a = S.image_grads(c["seed"], C, H, W, l1_scale=False, with_alpha=c["bg"])
    bgs = np.random.default_rng(c["seed"]).uniform(0, 1, (C, 3)).astype(np.float32) if c["bg"] else None
    o = oracle.Options(sh_degree=sc["sh_degree"], antialiased=c["aa"])
    gpu = U.run_gpu(sc, antialiased=c["aa"], v_img=v_img, v_alpha=v_a, backgrounds=bgs)
    ref = U.oracle_reference(sc, o, gpu, v_img, v_a, bgs)
    p = ref["proj"]
    assert np.array_equal(gpu["radii"], p["radii"])
    vis = p["radii"][..., 0] > 0
    sp = gpu["splats"]
    assert np.array_equal(sp[..., 0:2][vis], p["mean2d_f"][vis])
    assert np.array_equal(sp[..., 3][vis], p["depth_f"][vis])
    np.testing.assert_allclose(sp[..., 8:11][vis], p["rgb"][vis], rtol=1e-5, atol=1e-5)
    assert gpu["M"] == len(ref["keys"])
    assert np.array_equal(gpu["keys"], ref["keys"])
    assert np.array_equal(gpu["ids"], ref["ids"])
    assert np.array_equal(gpu["offsets"], ref["offsets"])
    U.assert_images(gpu, ref, label=f"sweep{c['seed']}")
    a = ref["amb"]
    assert a["ambiguous"] <= 1e-3 * a["pixels"] + 1, U.amb_report(ref)
    U.assert_grads(sc, gpu, ref, label=f"sweep{c['seed']}")
