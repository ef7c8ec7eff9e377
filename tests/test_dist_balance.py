"""Next row f4 on CPU: LPT assignment properties and the BalancedLayer
protocol (CSR slot all-gather, deterministic LPT, broadcast rounds) with the
gloo backend at world size 2 and 3 (uneven head counts)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_2502_20766_b200 import dist as D


def test_lpt_properties():
    rng = np.random.default_rng(3)
    for trial in range(50):
        H = int(rng.integers(1, 40))
        P = int(rng.integers(1, 9))
        costs = [int(x) for x in rng.integers(1, 1000, H)]
        a = D.lpt_assign(costs, P)
        assert sorted(h for x in a for h in x) == list(range(H))  # a partition
        loads = [sum(costs[h] for h in x) for x in a]
        # LPT guarantee (Graham): makespan <= 4/3 OPT, and OPT >= max(mean, max cost)
        lb = max(sum(costs) / P, max(costs))
        assert max(loads) <= 4 / 3 * lb + 1e-9
        assert a == D.lpt_assign(list(costs), P)  # deterministic
    # equal costs -> round-robin by index, ties to the lower rank
    assert D.lpt_assign([5, 5, 5, 5, 5], 2) == [[0, 2, 4], [1, 3]]
    assert D.head_cost(3, 2) == 4 * 128 * (128 * 128 * 1 + 2 * 128 * 129 // 2)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def fake_csr(h, nb):
    """deterministic per-head block rows with head-dependent density."""
    rows = []
    for qb in range(nb):
        ks = [kb for kb in range(qb + 1) if kb == 0 or kb == qb or (kb * 7 + h * 3 + qb) % (h % 4 + 2) == 0]
        rows.append(ks)
    return rows


def fake_out(h, rows, n, d):
    x = np.zeros((n, d), np.float32)
    for qb, ks in enumerate(rows):
        x[qb * 4:(qb + 1) * 4] = h * 1000 + qb * 10 + len(ks)
    return torch.from_numpy(x)


def _worker(rank, world, port, H, G, n, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b, d = 4, 3
        nb = -(-n // b)
        h0, h1 = D.head_range(H, world, rank)

        def plan_select(rp_slot, ci_slot):
            for i, h in enumerate(range(h0, h1)):
                rows = fake_csr(h, nb)
                off = 0
                rp_slot[i, 0] = 0
                for qb, ks in enumerate(rows):
                    ci_slot[i, off: off + len(ks)] = torch.tensor(ks, dtype=torch.int32)
                    off += len(ks)
                    rp_slot[i, qb + 1] = off

        out = torch.full((H, n, d), -1.0)

        def attend(h, rp, ci):
            rows = [ci[0, rp[0, qb]: rp[0, qb + 1]].tolist() for qb in range(nb)]
            assert rows == fake_csr(h, nb)  # the gathered CSR is the owner's
            out[h] = fake_out(h, rows, n, d)

        L = D.BalancedLayer(H, G, n, world, rank, plan_select, attend, "cpu", b=b)
        assign = L.step(out)
        exp = torch.stack([fake_out(h, fake_csr(h, nb), n, d) for h in range(H)])
        q.put((rank, bool(torch.equal(out, exp)), assign))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,H,G", [(2, 8, 2), (3, 7, 7)])
def test_balanced_layer_gloo(world, H, G):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n = 24
    ps = [ctx.Process(target=_worker, args=(r, world, port, H, G, n, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assigns = {tuple(map(tuple, a)) for _, _, a in res}
    assert len(assigns) == 1  # every rank computed the same assignment
    assert all(ok for _, ok, _ in res)  # every rank holds the full, correct output


def _worker_p2p(rank, world, port, H, G, n, outs, q):
    """exchange='p2p': each rank's attend stores its head into EVERY rank's
    buffer (shared-memory CPU tensors stand in for the NVLink-mapped peer
    buffers), then one barrier; no broadcast rounds."""
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b, d = 4, 3
        nb = -(-n // b)
        h0, h1 = D.head_range(H, world, rank)
        bases = [(r + 1) << 40 for r in range(world)]
        head_bytes = n * d * 2

        def plan_select(rp_slot, ci_slot):
            for i, h in enumerate(range(h0, h1)):
                rows = fake_csr(h, nb)
                off = 0
                rp_slot[i, 0] = 0
                for qb, ks in enumerate(rows):
                    ci_slot[i, off: off + len(ks)] = torch.tensor(ks, dtype=torch.int32)
                    off += len(ks)
                    rp_slot[i, qb + 1] = off

        seen = []

        def attend(h, rp, ci, peers):
            rows = [ci[0, rp[0, qb]: rp[0, qb + 1]].tolist() for qb in range(nb)]
            assert rows == fake_csr(h, nb)
            others = [r for r in range(world) if r != rank]
            assert peers.tolist() == [bases[r] + h * head_bytes for r in others]
            val = fake_out(h, rows, n, d)
            outs[rank][h] = val          # the kernel's own store
            for r in others:             # the fused peer stores
                outs[r][h] = val
            seen.append(h)

        L = D.BalancedLayer(H, G, n, world, rank, plan_select, attend, "cpu", b=b, exchange="p2p",
                            peer_bases=bases, head_bytes=head_bytes,
                            barrier=lambda: dist.barrier())
        assign = L.step(outs[rank])
        exp = torch.stack([fake_out(h, fake_csr(h, nb), n, d) for h in range(H)])
        q.put((rank, bool(torch.equal(outs[rank], exp)), assign, sorted(seen)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,H,G", [(2, 8, 2), (3, 7, 7)])
def test_balanced_layer_p2p_gloo(world, H, G):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n, d = 24, 3
    outs = [torch.full((H, n, d), -1.0).share_memory_() for _ in range(world)]
    ps = [ctx.Process(target=_worker_p2p, args=(r, world, port, H, G, n, outs, q))
          for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    assigns = {tuple(map(tuple, a)) for _, _, a, _ in res}
    assert len(assigns) == 1
    assign = list(assigns)[0]
    for rank, ok, _, seen in res:
        assert ok, rank                         # full output on every rank after the barrier
        assert seen == sorted(assign[rank])     # each rank computed exactly its LPT heads


def test_p2p_requires_peer_info():
    with pytest.raises(ValueError):
        D.BalancedLayer(4, 1, 16, 2, 0, None, None, "cpu", b=4, exchange="p2p")
    with pytest.raises(ValueError):
        D.BalancedLayer(4, 1, 16, 2, 0, None, None, "cpu", b=4, exchange="nvshmem")
