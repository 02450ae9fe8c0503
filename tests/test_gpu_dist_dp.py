"""Views-DP across real processes (the bench's --gpus N step): 2 and 3 ranks
under torch.distributed.run sharing this box's one GPU over gloo.  The all-reduced flat
gradient must equal the one-process multi-view gradient up to fp32 summation order, and the
oracle's gradient summed over all views with the parity contract."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

import oracle
from paper_2409_06765_b200 import dist as D
from synth import scenes as S
from tests import parity_util as U
from tests._dist_dp_worker import scene

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,mode", [(2, "flat"), (3, "flat"), (2, "bucketed"), (3, "bucketed")])
def test_views_dp_equals_one_process_and_oracle(tmp_path, world, mode):
    """flat: one all-reduce of the section-major flat gradient after the step; bucketed: the
    projection backward in 3 Gaussian buckets, each all-reduced asynchronously right after its
    kernel (DPEngine.backward_allreduce, the bench's N > 1 step)."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()),
           os.path.join(ROOT, "tests", "_dist_dp_worker.py"), str(tmp_path), mode]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    sc = scene()
    C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
    v_img, _ = S.image_grads(5, C, H, W, l1_scale=False)
    one = U.run_gpu(sc, v_img=v_img)
    seen = []
    for rk in range(world):
        vw = np.load(os.path.join(tmp_path, f"views{rk}.npy"))
        seen += list(vw)
        assert np.array_equal(np.load(os.path.join(tmp_path, f"rgb{rk}.npy")), one["rgb"][vw])
    assert sorted(seen) == list(range(C))
    if mode == "bucketed":
        dp = dict(np.load(os.path.join(tmp_path, "grads.npz")))
    else:
        flat = np.load(os.path.join(tmp_path, "flat.npy"))
        lay, _ = D.flat_layout(N, 16, True)
        dp = {"v_" + k: flat[o:o + n].reshape(shp) for k, (o, n, shp) in lay.items()}
    o = oracle.Options(sh_degree=3)
    ref = U.oracle_reference(sc, o, one, v_img, with_isect=False)
    # the all-reduced sum against the one-process call: the same per-(c,n) terms, another
    # summation order (camera partial sums added across ranks)
    U.assert_same_kernel_grads(sc, o, ref["bwd"], dp, one, label=f"dp{world}-vs-one")
    # and against the oracle's sum over all views
    U.assert_grads(sc, dp, ref, label=f"dp{world}", vs=one["v_splats"])
