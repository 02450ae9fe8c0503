"""Worker of tests/test_gpu_dist_api.py (run under torch.distributed.run): Gaussian-sharded
rasterization(distributed=True) on one GPU shared by all ranks (gloo backend; NCCL with one
rank, since NCCL takes one GPU per rank), one shard of
the scene and one block of cameras per rank; saves images and shard gradients to out_dir."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_06765_b200 import rasterization  # noqa: E402
from paper_2409_06765_b200 import dist as D  # noqa: E402
from paper_2409_06765_b200.gshard import shard_range  # noqa: E402
from synth import scenes as S  # noqa: E402


def main(out_dir, aa, backend="gloo"):
    if backend == "nccl":
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    dist.init_process_group(backend)
    rank, world = dist.get_rank(), dist.get_world_size()
    sc = S.tiny_scene(1, N=1500, width=200, height=150, sh_degree=3, views=3)
    C, N, W, H = 3, 1500, 200, 150
    n0, n1 = shard_range(N, world, rank)
    views = D.partition_views(C, world, rank)
    keys = ["means", "quats", "scales", "opacities", "colors"]
    g = [torch.from_numpy(np.ascontiguousarray(sc[k][n0:n1], np.float32)).cuda().requires_grad_(True) for k in keys]
    vm = torch.from_numpy(np.ascontiguousarray(sc["viewmats"][views], np.float32)).cuda()
    Ks = torch.from_numpy(np.ascontiguousarray(sc["Ks"][views], np.float32)).cuda()
    v, va = S.image_grads(3, C, H, W, l1_scale=False, with_alpha=True)
    rgb, alpha, meta = rasterization(*g, vm, Ks, W, H, sh_degree=3, distributed=True,
                                     rasterize_mode="antialiased" if aa else "classic")
    loss = (rgb * torch.from_numpy(v[views]).cuda()).sum() + (alpha[..., 0] * torch.from_numpy(va[views]).cuda()).sum()
    loss.backward()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), rgb=rgb.detach().cpu().numpy(),
             alpha=alpha.detach().cpu().numpy(), views=np.array(views, np.int64), n0=n0, n1=n1,
             **{f"g_{k}": t.grad.cpu().numpy() for k, t in zip(keys, g)})
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]), sys.argv[3] if len(sys.argv) > 3 else "gloo")
