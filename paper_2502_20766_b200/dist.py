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


# ------------------------------------------------ next row f4: balancing ----
def head_cost(nnz, nb, b=128, d=128):
    """Useful attention FLOPs of one head with `nnz` computed blocks (the
    diagonal blocks are half used): 4 d [b^2 (nnz - nb) + nb b (b+1)/2]."""
    return 4 * d * (b * b * (int(nnz) - nb) + nb * b * (b + 1) // 2)


def lpt_assign(costs, P):
    """Longest-processing-time-first assignment of heads to P ranks: heads in
    decreasing cost (ties -> lower head index) each go to the currently
    least-loaded rank (ties -> lower rank). Deterministic, so every rank
    computes the same assignment from the same (all-gathered) costs.
    Returns per-rank ascending head lists."""
    order = sorted(range(len(costs)), key=lambda h: (-costs[h], h))
    load = [0] * P
    out = [[] for _ in range(P)]
    for h in order:
        r = min(range(P), key=lambda i: (load[i], i))
        out[r].append(h)
        load[r] += costs[h]
    return [sorted(x) for x in out]


def imbalance(costs, assignment):
    """max over ranks of the assigned cost / mean cost (1.0 = perfect)."""
    loads = [sum(costs[h] for h in hs) for hs in assignment]
    mean = sum(loads) / len(loads)
    return max(loads) / mean if mean > 0 else 1.0


def static_assignment(H, P):
    return [list(range(*head_range(H, P, r))) for r in range(P)]


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
    return unpad_gathered(full, H, P)


def unpad_gathered(full, H, P):
    """[P * ceil(H/P)][n][d] all-gather result (rank r's slot holds its heads
    first, then padding) -> the [H][n][d] layer output in head order."""
    import torch
    hmax = max_heads(H, P)
    if hmax * P == H:
        return full
    idx = []
    for r in range(P):
        h0, h1 = head_range(H, P, r)
        idx.extend(range(r * hmax, r * hmax + (h1 - h0)))
    return full[torch.tensor(idx, device=full.device)]


class BalancedLayer:
    """Next row f4: cost-balanced (LPT) attention across ranks, with the output
    all-gather overlapped with the attention. Every rank holds the whole
    layer's Q/K/V (replicated inputs) and the full output buffer. One step:

      1. plan + select for this rank's static contiguous head range (the same
         split as the static partition), written into this rank's CSR slot;
      2. all-gather of the CSR slots (row_ptr [hmax][nb+1], col_idx
         [hmax][cap] per rank; NCCL over NVLink);
      3. per-head costs = useful attention FLOPs from row_ptr[:, nb], LPT
         assignment (deterministic, so every rank computes the same one). The
         costs of step t come from step t-1's gathered CSR, copied to pinned
         host memory asynchronously (no host synchronisation inside a step;
         only the first step reads its own CSR synchronously). Any assignment
         yields the same output (every head is computed exactly once and
         exchanged), so reusing the previous step's costs only affects balance;
      4. attention of this rank's LPT heads, one launch per head, each
         followed by an event on the compute stream;
      5. broadcast rounds j = 0, 1, ...: every rank broadcasts the output of
         its j-th head, issued on a communication stream after that head's
         event, so the exchange overlaps the remaining attention.

    exchange="p2p" (next row f4, the fused exchange): instead of step 5, the
    attention kernel's epilogue stores each output row into every rank's
    output buffer as well (fp_sparse_attn_peers over NVLink; the buffers are
    one symmetric-memory allocation whose peer base addresses are
    `peer_bases`), and one cross-rank barrier (`barrier`, stream-ordered on
    the GPU) ends the step. attend is then called as attend(h, rp, ci, peers)
    with `peers` the device table of the other ranks' head-h addresses
    (peer_table(h)), or None at one rank.

    The compute is injected (plan_select(rp_slot, ci_slot), attend(h, rp, ci))
    so the protocol is testable with the gloo backend on CPU tensors.
    """

    def __init__(self, H, G, n, world, rank, plan_select, attend, device, group=None, b=128,
                 exchange="nccl", peer_bases=None, head_bytes=None, barrier=None):
        import torch
        self.H, self.G, self.n, self.P, self.rank = H, G, n, world, rank
        self.nb = -(-n // b)
        self.cap = self.nb * (self.nb + 1) // 2
        self.hmax = max_heads(H, world)
        self.ranges = [head_range(H, world, r) for r in range(world)]
        self.plan_select, self.attend = plan_select, attend
        self.device, self.group = torch.device(device), group
        i32 = torch.int32
        self.rp_slot = torch.zeros((self.hmax, self.nb + 1), dtype=i32, device=device)
        self.ci_slot = torch.zeros((self.hmax, self.cap), dtype=i32, device=device)
        self.rp_all = torch.empty((world * self.hmax, self.nb + 1), dtype=i32, device=device)
        self.ci_all = torch.empty((world * self.hmax, self.cap), dtype=i32, device=device)
        self.cuda = self.device.type == "cuda"
        self.comm = torch.cuda.Stream(device=self.device) if self.cuda else None
        self.last_assignment = None
        self.last_costs = None
        self._nnz_host = None  # previous step's per-slot nnz (pinned, async copy)
        self._nnz_event = None
        if exchange not in ("nccl", "p2p"):
            raise ValueError(exchange)
        self.exchange = exchange
        self.barrier = barrier
        self.peer_tab = None
        if exchange == "p2p":
            if barrier is None or head_bytes is None or peer_bases is None or len(peer_bases) != world:
                raise ValueError("exchange='p2p' needs peer_bases (one per rank), head_bytes, barrier")
            others = [r for r in range(world) if r != rank]
            # row h: the other ranks' addresses of head h (device int64 table)
            tab = [[int(peer_bases[r]) + h * int(head_bytes) for r in others] for h in range(H)]
            self.peer_tab = torch.tensor(tab, dtype=torch.int64, device=device) if others else None

    def peer_table(self, h):
        """device int64 [P-1] of the other ranks' output addresses of head h (p2p), or None"""
        return None if self.peer_tab is None else self.peer_tab[h]

    def slot(self, h):
        """row of rp_all / ci_all holding head h's CSR."""
        for r, (h0, h1) in enumerate(self.ranges):
            if h0 <= h < h1:
                return r * self.hmax + (h - h0)
        raise IndexError(h)

    def step(self, out, timers=None):
        import torch
        import torch.distributed as dist
        stream = torch.cuda.current_stream(self.device) if self.cuda else None

        def mark(key):
            if timers is not None and self.cuda:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(stream)
                timers.setdefault(key, []).append(ev)

        mark("t0")
        self.plan_select(self.rp_slot, self.ci_slot)
        mark("t1")
        dist.all_gather_into_tensor(self.rp_all, self.rp_slot, group=self.group)
        dist.all_gather_into_tensor(self.ci_all, self.ci_slot, group=self.group)
        if self._nnz_host is None:
            nnz = self.rp_all[:, self.nb].cpu().tolist()  # first step: read synchronously
        else:
            if self._nnz_event is not None:
                self._nnz_event.synchronize()  # the previous step's copy: long complete
            nnz = self._nnz_host.tolist()
        if self.cuda:  # this step's costs, for the next step's assignment
            if self._nnz_host is None:
                self._nnz_host = torch.empty(self.P * self.hmax, dtype=torch.int32).pin_memory()
            self._nnz_host.copy_(self.rp_all[:, self.nb], non_blocking=True)
            self._nnz_event = torch.cuda.Event()
            self._nnz_event.record(stream)
        else:
            self._nnz_host = self.rp_all[:, self.nb].clone()
        costs = [head_cost(nnz[self.slot(h)], self.nb) for h in range(self.H)]
        assign = lpt_assign(costs, self.P)
        self.last_assignment, self.last_costs = assign, costs
        mark("t2")
        mine = assign[self.rank]
        if self.exchange == "p2p":
            # fused exchange: every launch also stores its rows into the peers'
            # buffers; one barrier after the last launch completes the layer
            for h in mine:
                s = self.slot(h)
                self.attend(h, self.rp_all[s: s + 1], self.ci_all[s: s + 1], self.peer_table(h))
            mark("t3")
            self.barrier()
            mark("t4")
            return assign
        events = []
        for h in mine:
            s = self.slot(h)
            self.attend(h, self.rp_all[s: s + 1], self.ci_all[s: s + 1])
            if self.cuda:
                ev = torch.cuda.Event()
                ev.record(stream)
                events.append(ev)
        mark("t3")
        rounds = max(len(x) for x in assign)
        if self.cuda:
            self.comm.wait_stream(stream) if not events else None
            ctx = torch.cuda.stream(self.comm)
        else:
            import contextlib
            ctx = contextlib.nullcontext()
        with ctx:
            for j in range(rounds):
                if self.cuda and j < len(events):
                    self.comm.wait_event(events[j])
                for r in range(self.P):
                    if j < len(assign[r]):
                        dist.broadcast(out[assign[r][j]], src=r, group=self.group)
        if self.cuda:
            stream.wait_stream(self.comm)
        mark("t4")
        return assign
