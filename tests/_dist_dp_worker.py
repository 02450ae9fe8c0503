"""Worker of tests/test_gpu_dist_dp.py (run under torch.distributed.run): the views-DP step
of bench.py / SURVEY 8(e) -- Gaussians replicated, this rank's contiguous block of views
rendered by one Engine call, the flat parameter gradient summed with ONE all-reduce.  Ranks
share the box's one GPU over gloo (NCCL takes one GPU per rank).  Rank 0 saves the summed
flat gradient; every rank saves its images."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2409_06765_b200.engine import DPEngine, Engine  # noqa: E402
from paper_2409_06765_b200 import dist as D  # noqa: E402
from synth import scenes as S  # noqa: E402


def scene():
    return S.mipnerf_like_scene(20000, width=320, height=200, views=4, sh_degree=3, seed=31)


def main(out_dir, bucketed=False):
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    sc = scene()
    C, N, W, H = sc["viewmats"].shape[0], sc["means"].shape[0], sc["width"], sc["height"]
    views = D.partition_views(C, world, rank)
    v_img, _ = S.image_grads(5, C, H, W, l1_scale=False)
    keys = ["means", "quats", "scales", "opacities", "colors"]
    dev = torch.device("cuda", 0)
    params = [torch.from_numpy(np.ascontiguousarray(sc[k], np.float32)).to(dev) for k in keys]
    params += [torch.from_numpy(np.ascontiguousarray(sc[k][views], np.float32)).to(dev) for k in ("viewmats", "Ks")]
    v = torch.from_numpy(np.ascontiguousarray(v_img[views])).to(dev)
    if bucketed:
        # the bench's N > 1 step: projection backward in buckets, each bucket all-reduced
        # asynchronously right after its kernel (gloo takes the CUDA tensors here)
        eng = DPEngine(N, len(views), W, H, sh_degree=3, device=dev, buckets=3)
        eng.run_checked(tuple(params), v)
        eng.forward(*params)
        eng.rasterize_bwd(v)
        eng.backward_allreduce(tuple(params))
        torch.cuda.synchronize()
        flat = dict((k, t.cpu()) for k, t in eng.grads().items())
    else:
        eng = Engine(N, len(views), W, H, sh_degree=3, device=dev)
        eng.run_checked(tuple(params), v)
        torch.cuda.synchronize()
        flat = eng.flat_grad.cpu()            # the collective runs on the host buffer over gloo
        D.allreduce_grads(flat)
    np.save(os.path.join(out_dir, f"rgb{rank}.npy"), eng.out_rgb.cpu().numpy())
    np.save(os.path.join(out_dir, f"views{rank}.npy"), np.array(views, np.int64))
    if rank == 0:
        if bucketed:
            np.savez(os.path.join(out_dir, "grads.npz"), **{k: t.numpy() for k, t in flat.items()})
        else:
            np.save(os.path.join(out_dir, "flat.npy"), flat.numpy())
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(sys.argv[1], len(sys.argv) > 2 and sys.argv[2] == "bucketed")
