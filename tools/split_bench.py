"""Single-transform loop split across GPUs: time one large
ATSFFT with its estimation loops split over the ranks (c5-style: 16384^2,
b_estimate 8192, 8 loops) or one SFFT with location + estimation loops split.

  torchrun --nproc-per-node N --master-addr 127.0.0.1 tools/split_bench.py \
      [--algo ats|sfft] [--side 16384] [--k 64] [--snr 15] [--reps 3]

Rank 0 prints one JSON line: ms per transform (max over ranks, CUDA events on
each rank's stream around the whole call incl. its collectives) and whether the
result equals the single-GPU path."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1908_02461_b200 as P  # noqa: E402
from paper_1908_02461_b200 import distributed as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--algo", choices=["ats", "sfft"], default="ats")
    ap.add_argument("--side", type=int, default=16384)
    ap.add_argument("--k", type=int, default=64)
    ap.add_argument("--snr", type=float, default=15.0)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--precision", default="fp32")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ.setdefault("MASTER_PORT", "29533")
    dist.init_process_group("nccl", rank=rank, world_size=world)
    img = P.sparse_image(args.side, args.k, 5, snr_db=args.snr, cluster_frac=0.2)
    x = torch.from_numpy(img.x).cuda()
    if args.algo == "ats":
        run = lambda: D.atsfft2d_loopsplit(x, P.TunerConfig(), 8, 11, precision=args.precision)[0]  # noqa: E731
        single = lambda: P.atsfft2d(x, P.TunerConfig(), 8, 11, precision=args.precision)[0]  # noqa: E731
    else:
        cfg = P.SfftConfig(n=args.side, k=args.k)
        run = lambda: D.sfft2d_loopsplit(x, cfg, 11, precision=args.precision)  # noqa: E731
        single = lambda: P.sfft2d(x, cfg, 11, precision=args.precision)  # noqa: E731
    out = run()
    same = None
    if rank == 0:
        ref = single()
        same = set(out) == set(ref)
    times = []
    for _ in range(args.reps):
        dist.barrier(device_ids=[local])
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        run()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        times.append(float(t.item()))
    if rank == 0:
        print(json.dumps({"algo": args.algo, "n": args.side, "k": args.k, "gpus": world,
                          "ms_per_transform": float(np.median(times)), "samples_ms": times,
                          "support_equal_to_single_gpu": same, "precision": args.precision}))
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
