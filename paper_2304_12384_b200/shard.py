"""Frame-range sharding across GPUs.

Frames are independent except for h, which couples frame t to t-1 (S:218-226,
S:362).  Rank r of N owns the contiguous POC range
[r*F/N, (r+1)*F/N) and additionally analyses the frame just before it as a
one-frame halo (vca_analyze n_halo = 1), so every rank's first h is taken
against the true previous frame and the records are bit-identical to an
unsharded run.  The only collective is one all-gather of the 64-byte
per-frame records (NCCL over NVLink on the GPU; gloo in the CPU tests).
This module is host logic only: plans, padding and the gather.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    world: int
    first_poc: int     # first emitted POC of this rank
    count: int         # records this rank emits
    first_frame: int   # first frame this rank reads (first_poc - n_halo)
    n_frames: int      # frames this rank analyses (count + n_halo)
    n_halo: int        # 1 if a halo frame precedes the range, else 0


def plan(n_total: int, world: int, rank: int, halo: bool = True) -> Shard:
    """Contiguous split of POCs 0..n_total-1 over `world` ranks (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world or n_total < world:
        raise ValueError("need 0 <= rank < world <= n_total")
    first = rank * n_total // world
    last = (rank + 1) * n_total // world
    n_halo = 1 if (halo and first > 0) else 0
    return Shard(rank, world, first, last - first, first - n_halo, last - first + n_halo, n_halo)


def gather_records(local, world: int, group=None, counts=None):
    """All-gather per-rank record tensors [count_r, 8] (float64 views of vca_features)
    into one [sum count_r, 8] tensor in rank (= POC) order.  Uneven counts are padded
    to the maximum for the collective and trimmed after.  `counts` (per-rank record
    counts, e.g. from plan()) skips the count exchange."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return local
    if counts is None:
        n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
        cnt = [torch.zeros_like(n) for _ in range(world)]
        dist.all_gather(cnt, n, group=group)
        counts = [int(c.item()) for c in cnt]
    m = max(counts)
    pad = local
    if local.shape[0] < m:
        pad = torch.zeros((m, local.shape[1]), dtype=local.dtype, device=local.device)
        pad[: local.shape[0]] = local
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * m, local.shape[1]), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, pad.contiguous(), group=group)
        parts = [out[i * m: i * m + counts[i]] for i in range(world)]
    else:  # gloo: host tensors
        host = pad.detach().cpu().contiguous()
        bufs = [torch.empty_like(host) for _ in range(world)]
        dist.all_gather(bufs, host, group=group)
        parts = [bufs[i][: counts[i]].to(local.device) for i in range(world)]
    return torch.cat(parts, dim=0)
