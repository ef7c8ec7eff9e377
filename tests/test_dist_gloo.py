"""Multi-rank head partition + output all-gather, on CPU with gloo (world 2).

The per-rank compute is the float64 oracle on that rank's head slice (the
GPU path is not available here); the test checks that the partition covers
every head exactly once, that every segment is launchable with a uniform GQA
mapping, and that the gathered output equals the single-process result
bitwise (heads are independent, so the partition cannot change any value).
"""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_20766_b200 import dist as fpdist


@pytest.mark.parametrize("H,G,P", [(32, 8, 8), (32, 2, 4), (28, 4, 8), (32, 4, 8), (28, 4, 3),
                                   (4, 1, 2), (7, 7, 2)])
def test_partition_covers_heads_once(H, G, P):
    seen = []
    for h0, h1, segs in fpdist.partition(H, G, P):
        assert h1 - h0 in (H // P, -(-H // P))
        covered = []
        for s in segs:
            covered.extend(range(s.h0, s.h1))
            hs, gs = s.h1 - s.h0, s.g1 - s.g0
            assert hs % gs == 0
            for h in range(s.h0, s.h1):  # uniform local GQA mapping == global mapping
                assert s.g0 + (h - s.h0) * gs // hs == h * G // H
        assert covered == list(range(h0, h1))
        seen.extend(covered)
    assert seen == list(range(H))


def _worker(rank, world, port, H, G, n, q, k, v, ref, q_out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        h0, h1, segs = fpdist.partition(H, G, world)[rank]
        local = torch.zeros((h1 - h0, n, 128), dtype=torch.float64)
        for s in segs:
            for h in range(s.h0, s.h1):
                g = h * G // H
                r = oracle.flexprefill_head(q[h], k[g], v[g], 128, 0.9, 0.1, 0)
                local[h - h0] = torch.from_numpy(r["out"])
        full = fpdist.gather_heads(local, H, world)
        q_out.put((rank, bool(torch.equal(full, torch.from_numpy(ref)))))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_gather_equals_single_process():
    from synth import gen
    from synth.configs import Workload
    import oracle
    H, G, n = 7, 1, 512  # uneven: ranks get 4 and 3 heads
    w = Workload("dist", H, G, n, 0.9, 0.1, 0, 21)
    qb, kb, vb = gen.make_layer_bits(w)
    q, k, v = (gen.bits_to_f64(x) for x in (qb, kb, vb))
    ref = np.stack([oracle.flexprefill_head(q[h], k[0], v[0], 128, 0.9, 0.1, 0)["out"]
                    for h in range(H)])
    ctx = mp.get_context("spawn")
    qo = ctx.Queue()
    port = 29500 + (os.getpid() % 1000)
    procs = [ctx.Process(target=_worker, args=(r, 2, port, H, G, n, q, k, v, ref, qo))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = sorted(qo.get(timeout=5) for _ in range(2))
    assert res == [(0, True), (1, True)]
