"""K7 visit statistics (debug build only): run on a GPU box as

    GS_NVCC_EXTRA=-DGS_K7_STATS python -m paper_2409_06765_b200.build --force && python tools/k7_stats.py

It renders BASELINE configs[1] and prints K7's (warp, splat) visit counts: empty visits,
contributing lanes per visit, few-lane vs shuffle-tree reductions, visits where only one
4x4 half of the 8x4 warp takes the splat.  (The normal build has no counters.)"""
import ctypes as ct, numpy as np, torch, sys
sys.path.insert(0, '.')
from paper_2409_06765_b200 import Engine, _lib as L
from synth import scenes as S
sc = S.scene_from_config('garden1m')
C, N, W, H = 1, sc['means'].shape[0], sc['width'], sc['height']
keys = ["means", "quats", "scales", "opacities", "colors", "viewmats", "Ks"]
params = tuple(torch.from_numpy(np.ascontiguousarray(sc[k], np.float32)).cuda() for k in keys)
v_img, _ = S.image_grads(1002, 1, H, W)
v = torch.from_numpy(v_img).cuda()
lib = L.lib()
f = lib.gs_debug_k7_stats; f.restype = ct.c_int; f.argtypes = [ct.c_void_p, ct.c_int]
for mode in (0, 2):
    e = Engine(N, C, W, H, sh_degree=3, bbox_mode=mode)
    e.run_checked(params, v)
    torch.cuda.synchronize()
    buf = (ct.c_ulonglong * 8)()
    f(buf, 1)
    e.rasterize_bwd(v)
    torch.cuda.synchronize()
    f(buf, 0)
    s = list(buf)
    print(f"bbox{mode}: visits {s[0]/1e6:.2f}M empty {s[1]/1e6:.2f}M ({s[1]/s[0]:.1%}) lanes/visit(nonempty) {s[2]/(s[0]-s[1]):.2f} "
          f"few {s[3]/1e6:.2f}M tree {(s[0]-s[1]-s[3])/1e6:.2f}M one-half-only {s[4]/1e6:.2f}M  contributing pairs {s[2]/1e6:.1f}M")
    ne = s[0] - s[1]
    print(f"   per non-empty visit: lanes inside {s[7]/ne:.2f}, alive (tidx <= last) {s[5]/ne:.2f}, "
          f"in support (alpha >= alpha_min) {s[6]/ne:.2f}, contributing {s[2]/ne:.2f}")
