"""rasterization(distributed=True) (NEXT-4(i)) across real processes: 2 and 3 ranks
under torch.distributed.run sharing this box's one GPU over gloo (the product uses NCCL with
one GPU per rank; the collectives' semantics are the same).  Images of every rank's cameras
must be bit-identical to the one-process call over the whole scene, and the concatenated
shard gradients equal to its gradients up to fp32 atomic order.  The NCCL case (one rank:
NCCL cannot put two ranks on one GPU) runs the same path with device-side collectives."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

from synth import scenes as S
from tests import parity_util as U

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,aa,backend", [(2, 0, "gloo"), (3, 1, "gloo"), (1, 0, "nccl")])
def test_distributed_rasterization_matches_one_process(tmp_path, world, aa, backend):
    import torch
    from paper_2409_06765_b200 import rasterization
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "_dist_raster_worker.py"), str(tmp_path), str(aa), backend]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    sc = S.tiny_scene(1, N=1500, width=200, height=150, sh_degree=3, views=3)
    C, N, W, H = 3, 1500, 200, 150
    ts = [t.clone().requires_grad_(i < 5) for i, t in enumerate(U.to_torch(sc, "cuda"))]
    rgb, alpha, _ = rasterization(*ts, W, H, sh_degree=3, rasterize_mode="antialiased" if aa else "classic")
    v, va = S.image_grads(3, C, H, W, l1_scale=False, with_alpha=True)
    loss = (rgb * torch.from_numpy(v).cuda()).sum() + (alpha[..., 0] * torch.from_numpy(va).cuda()).sum()
    loss.backward()
    rgb, alpha = rgb.detach().cpu().numpy(), alpha.detach().cpu().numpy()
    keys = ["means", "quats", "scales", "opacities", "colors"]
    grads = {k: np.zeros_like(t.grad.cpu().numpy()) for k, t in zip(keys, ts)}
    seen = []
    for rk in range(world):
        d = np.load(os.path.join(tmp_path, f"rank{rk}.npz"))
        vw = d["views"]
        seen += list(vw)
        assert np.array_equal(d["rgb"], rgb[vw]) and np.array_equal(d["alpha"], alpha[vw])
        for k in keys:
            grads[k][int(d["n0"]):int(d["n1"])] = d[f"g_{k}"]
    assert sorted(seen) == list(range(C))
    # same kernels in another fp32 atomic order: within the atomic-order bound
    import oracle
    o = oracle.Options(sh_degree=3, antialiased=aa)
    b = oracle.render_bwd(oracle.project(sc, o), C, N, W, H, o, v.astype(np.float64), va.astype(np.float64))
    U.assert_same_kernel_grads(sc, o, b, {"v_" + k: g for k, g in grads.items()},
                               {"v_" + k: t.grad.cpu().numpy() for k, t in zip(keys, ts)}, label=f"dist{world}")
