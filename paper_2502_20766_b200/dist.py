"""Head partitioning across ranks.

Heads are independent units of work (the method adapts to "each
input and attention head"); the only coupling is GQA's read-only sharing of
K/V. Rank r gets a contiguous, balanced range of Q heads (the first H mod P
ranks get one extra head) plus the KV heads those Q heads read. The only
exchange step is the all-gather of the bf16 outputs (torch.distributed /
NCCL over NVLink); plan, select and attention need no communication.
"""
from dataclasses import dataclass


@dataclass(frozen=True)
class Segment:
    """A run of Q heads [h0, h1) of one rank that can be launched as one
    C-ABI call: local heads h0..h1-1 map onto KV heads [g0, g1) with uniform
    group size (h - h0) * (g1 - g0) // (h1 - h0) + g0 == h * G // H."""
    h0: int
    h1: int
    g0: int
    g1: int


def head_range(H, P, r):
    base, extra = divmod(H, P)
    h0 = r * base + min(r, extra)
    return h0, h0 + base + (1 if r < extra else 0)


def segments(H, G, h0, h1):
    """Split Q heads [h0, h1) into launchable segments (see Segment)."""
    g = H // G
    if h1 <= h0:
        return []
    if h0 % g == 0 and (h1 - h0) % g == 0:
        return [Segment(h0, h1, h0 // g, h1 // g)]  # whole KV groups: one call
    out = []
    h = h0
    while h < h1:
        grp = h // g
        e = min(h1, (grp + 1) * g)
        out.append(Segment(h, e, grp, grp + 1))
        h = e
    return out


def partition(H, G, P):
    """Per-rank (h0, h1, [segments])."""
    res = []
    for r in range(P):
        h0, h1 = head_range(H, P, r)
        res.append((h0, h1, segments(H, G, h0, h1)))
    return res


def max_heads(H, P):
    return -(-H // P)


def gather_heads(local_out, H, P, group=None):
    """All-gather each rank's [h1-h0][n][d] output slot (padded to ceil(H/P)
    heads) into the full [H][n][d] layer output (torch.distributed)."""
    import torch
    import torch.distributed as dist
    hmax = max_heads(H, P)
    n, d = local_out.shape[1], local_out.shape[2]
    if local_out.shape[0] != hmax:
        pad = torch.zeros((hmax, n, d), dtype=local_out.dtype, device=local_out.device)
        pad[: local_out.shape[0]] = local_out
        local_out = pad
    full = torch.empty((P * hmax, n, d), dtype=local_out.dtype, device=local_out.device)
    dist.all_gather_into_tensor(full, local_out.contiguous(), group=group)
    if hmax * P == H:
        return full
    idx = []
    for r in range(P):
        h0, h1 = head_range(H, P, r)
        idx.extend(range(r * hmax, r * hmax + (h1 - h0)))
    return full[torch.tensor(idx, device=full.device)]
