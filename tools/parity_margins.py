"""Measures how much of each parity tolerance the GPU path uses (B200): per scene, the
ambiguous-pixel statistics, the largest image / T error over ALL pixels (ambiguous ones
resolved to the outcome the GPU took), and the smallest floor factors the 2D and 3D gradient
checks would need.  Prints one JSON line per scene.  Test infrastructure (runs the oracle)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from synth import scenes as S  # noqa: E402
from tests import parity_util as U  # noqa: E402


def scene(name):
    if name == "tiny":
        return S.tiny_scene(0), 0, None
    if name == "tiny_sh3_ragged":
        return S.tiny_scene(1, N=1500, width=200, height=150, sh_degree=3, views=2), 0, None
    if name == "mip_small":
        return S.mipnerf_like_scene(20000, width=320, height=200, views=2, sh_degree=3, seed=11), 0, None
    if name == "mip_small_aa":
        return S.mipnerf_like_scene(20000, width=320, height=200, views=2, sh_degree=3, seed=12), 1, None
    if name == "rgb_direct":
        return S.tiny_scene(2, N=400, width=97, height=61, sh_degree=-1, views=3), 0, None
    if name == "garden1m":
        sc = S.scene_from_config("garden1m")
        return sc, 0, S.tile_subset_mask(0, 1, sc["width"], sc["height"], 32)
    raise KeyError(name)


def main(names):
    for name in names:
        sc, aa, mask = scene(name)
        C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
        v_img, _ = S.image_grads(0, C, H, W, l1_scale=False)
        if mask is not None:
            pm = np.repeat(np.repeat(mask, 16, 1), 16, 2)[:, :H, :W]
            v_img *= pm[..., None]
        o = oracle.Options(sh_degree=sc["sh_degree"], antialiased=aa)
        gpu = U.run_gpu(sc, antialiased=aa, v_img=v_img)
        ref = U.oracle_reference(sc, o, gpu, v_img, tile_mask=mask, with_isect=False)
        f, b, p = ref["fwd"], ref["bwd"], ref["proj"]
        sel = np.ones((C, H, W), bool) if mask is None else pm.astype(bool)
        out = dict(scene=name, amb=ref["amb"],
                   img_err=float(np.abs(gpu["rgb"] - f["rgb"])[sel].max()),
                   T_err=float(np.abs(gpu["T"] - f["T"])[sel].max()),
                   last_equal=bool(np.array_equal(U.last_gid(gpu, N)[sel], f["last_gid"][sel])))
        vis = p["radii"][..., 0] > 0
        g2 = U.v2d_from_splats(gpu["v_splats"])
        r2 = b["v2d"]
        exc = np.abs(g2 - r2) - U.GRAD_RTOL * np.abs(r2) - U.GRAD2D_ULP * b["s2d"] - b["d2d"]
        need = np.where(b["a2d"] > 0, exc / np.maximum(b["a2d"], 1e-300), np.where(exc > 0, np.inf, 0))[vis]
        out["grad2d_floor_needed"] = float(need.max())
        full = np.where(vis[..., None], np.where(b["a2d"] > 0, exc / np.maximum(b["a2d"], 1e-300), 0), -1)
        wi = np.unravel_index(int(np.argmax(full)), full.shape)
        out["grad2d_worst"] = dict(idx=[int(x) for x in wi], g=float(g2[wi]), r=float(r2[wi]), a=float(b["a2d"][wi]),
                                   s=float(b["s2d"][wi]), d=float(b["d2d"][wi]), n2d=int(b["n2d"][wi[:2]]),
                                   g_ambig=int(b["g_ambig"][wi[:2]]))
        out["grad2d_floor_p9999"] = float(np.quantile(need, 0.9999))
        # atomic-order model: need / (n2d u)
        n2d = np.maximum(b["n2d"], 1)[..., None] * np.ones_like(r2)
        out["grad2d_need_over_n_u"] = float((need / (n2d[vis] * 2.0 ** -24)).max())
        floors = U.grad3d_tolerance(sc, p, o, b)
        import oracle as O
        Ba = O.project_bwd_bound(sc, p, np.abs(r2), o)
        Bf = O.project_bwd_bound(sc, p, U.GRAD2D_FLOOR * b["a2d"] + U.GRAD2D_ULP * b["s2d"] + b["d2d"], o)
        Bc = O.project_bwd_clamp_alt(sc, p, r2, o)
        out["d2d_nonzero"] = int((b["d2d"] > 0).sum())
        out["clamp_alt_nonzero"] = int((Bc["v_colors"] > 0).sum())
        for k in ["v_means", "v_quats", "v_scales", "v_opacities", "v_colors"]:
            g, r = np.asarray(gpu[k], np.float64), ref["grads"][k]
            e = np.abs(g - r) - U.GRAD_RTOL * np.abs(r) - Bf[k] - Bc[k]
            nd = np.where(Ba[k] > 0, e / np.maximum(Ba[k], 1e-300), np.where(e > 0, np.inf, 0))
            nbad, worst, rel = U.check_grad3d_elementwise(g, r, floors[k])
            out[k] = dict(eps_needed=float(nd.max()), bad=nbad, worst_ratio=worst, rel=rel)
            if nbad:
                wi = np.unravel_index(int(np.argmax(nd)), nd.shape)
                out[k]["worst"] = dict(idx=[int(x) for x in wi], g=float(g[wi]), r=float(r[wi]),
                                       floor=float(floors[k][wi]), Ba=float(Ba[k][wi]))
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["tiny", "tiny_sh3_ragged", "mip_small", "mip_small_aa", "rgb_direct", "garden1m"])
