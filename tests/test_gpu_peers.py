"""Next row f4: the output exchange fused into the attention
epilogue (fp_sparse_attn_peers). On one GPU the "peer" buffers are further
local buffers: every one must receive exactly the rows the plain call writes
(bitwise), in plain and token-major layouts and for ragged n; rows past n and
heads outside the call stay untouched. Over NVLink the same stores target
other ranks' buffers mapped into the process (torch symmetric memory).
"""
import numpy as np
import pytest

from synth import gen
from synth.configs import Workload
from tests import parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fp():
    import paper_2502_20766_b200 as m
    m.load_library()
    return m


@pytest.mark.parametrize("n,layout", [(2048, None), (2085, None), (1000, "bshd")])
def test_peer_outputs_bitwise(fp, n, layout):
    import torch
    H, G = 8, 2
    w = Workload(f"peers-{n}", H, G, n, 0.9, 0.1, 0, 70 + n % 13)
    q, k, v = (parity.to_torch_bf16(x) for x in gen.make_layer_bits(w))
    if layout == "bshd":
        q, k, v = (x.transpose(0, 1).contiguous()[None] for x in (q, k, v))
    fpl = fp.FlexPrefill(H, G, n, layout=layout or "bhsd")
    fpl.plan(q, k, w.tau)
    fpl.select(w.gamma, 0)
    ref = torch.zeros_like(q)
    fpl.attn(q, k, v, ref)
    fill = torch.full_like(q, 3.0)
    outs = [fill.clone() for _ in range(3)]
    if layout == "bshd":  # a padded peer buffer: rows >= n must stay untouched
        outs = [torch.full((1, n + 24, H, 128), 3.0, dtype=torch.bfloat16, device="cuda")
                for _ in range(3)]
    ptrs = torch.tensor([o.data_ptr() for o in outs[1:]], dtype=torch.int64, device="cuda")
    fp.fp_sparse_attn_peers(q, k, v, outs[0], ptrs, 2, H, G, n, fpl.row_ptr, fpl.col_idx,
                            layout=fpl.layout, ws=fpl.ws, ws_bytes=fpl.ws_bytes)
    torch.cuda.synchronize()
    for o in outs:
        got = o[:, :n] if layout == "bshd" else o
        assert torch.equal(got, ref)
        if layout == "bshd":
            assert torch.all(o[:, n:] == 3.0)


def test_peer_outputs_single_head_slices(fp):
    """the multi-GPU LPT layer launches one head at a time into slices of the
    full output: peer pointers at a head offset must land on that head only."""
    import torch
    H, G, n = 4, 1, 2048
    w = Workload("peers-slices", H, G, n, 0.9, 0.1, 0, 77)
    q, k, v = (parity.to_torch_bf16(x) for x in gen.make_layer_bits(w))
    fpl = fp.FlexPrefill(H, G, n)
    fpl.plan(q, k, w.tau)
    fpl.select(w.gamma, 0)
    ref = torch.zeros_like(q)
    fpl.attn(q, k, v, ref)
    full = [torch.full_like(q, 5.0) for _ in range(2)]
    h = 2
    ptrs = torch.tensor([full[1][h].data_ptr()], dtype=torch.int64, device="cuda")
    rp, ci = fpl.row_ptr[h: h + 1].contiguous(), fpl.col_idx[h: h + 1].contiguous()
    fp.fp_sparse_attn_peers(q[h: h + 1], k[0: 1], v[0: 1], full[0][h: h + 1], ptrs, 1, 1, 1, n,
                            rp, ci)
    torch.cuda.synchronize()
    for f in full:
        assert torch.equal(f[h], ref[h])
        for hh in range(H):
            if hh != h:
                assert torch.all(f[hh] == 5.0)
    assert np.isfinite(ref.float().cpu().numpy()).all()
