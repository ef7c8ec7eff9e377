"""Next row f3: shape generality on the GPU.

* ragged n (n % 128 != 0, reading A26): full parity against the oracle,
  gamma = 1 bitwise equal to the dense kernel, min budget, host e2e path;
* fp_layout: token-major [batch][seq][heads][128] (the layout of a QKV
  projection) and batch > 1 give BITWISE the results of the plain head-major
  batch-1 calls on the same values (same kernels, only addressing differs).
"""
import numpy as np
import pytest

from synth import gen
from synth.configs import Workload
from tests import parity
from tests.test_gpu_parity import full_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fp():
    import paper_2502_20766_b200 as m
    m.load_library()
    return m


@pytest.mark.parametrize("heads,kv,n,gamma,min_budget", [
    (4, 1, 129, 0.9, 0),        # one-row last block; Q^ spans blocks 0 and 1
    (4, 2, 1000, 0.9, 0),       # last block 104 rows
    (8, 2, 2085, 0.95, 1024),   # last block 37 rows, min budget on
    (8, 2, 4301, 0.9, 0),       # 34 blocks: ragged last representative chunk as well
])
def test_ragged_full_parity(fp, heads, kv, n, gamma, min_budget):
    w = Workload(f"ragged-{n}", heads, kv, n, gamma, 0.1, min_budget, 31 + n % 97)
    res = full_parity(fp, w)
    nb = -(-n // 128)
    assert res["row_ptr"].shape[1] == nb + 1
    assert all(s_["nnz_blocks"] >= 2 * nb - 1 for s_ in res["stats"])  # forced blocks


def test_ragged_gamma_one_equals_dense(fp):
    w = Workload("ragged-g1", 4, 1, 1000, 1.0, 0.1, 0, 41)
    q, k, v = gen.make_layer_bits(w)
    res = parity.run_gpu(fp, w, q, k, v, gamma=1.0, dense=True)
    nb = 8
    assert np.all(res["row_ptr"][:, -1] == nb * (nb + 1) // 2)
    assert np.array_equal(res["out"], res["dense"])


def test_ragged_layer_host_matches_device_path(fp):
    import torch
    w = Workload("ragged-host", 8, 2, 2085, 0.9, 0.1, 0, 43)
    q, k, v = gen.make_layer_bits(w)
    res = parity.run_gpu(fp, w, q, k, v)
    fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
    qh, kh, vh = (torch.from_numpy(x).view(torch.bfloat16).pin_memory() for x in (q, k, v))
    oh = torch.empty_like(qh).pin_memory()
    dq, dk, dv = (torch.empty(x.shape, dtype=torch.bfloat16, device="cuda") for x in (qh, kh, vh))
    do = torch.empty_like(dq)
    fp.fp_layer_host(qh, kh, vh, oh, dq, dk, dv, do, w.heads, w.kv_heads, w.seq_len, w.gamma, w.tau,
                     0, fpl.ws, fpl.ws_bytes, fpl.pattern, fpl.jsd, fpl.row_ptr, fpl.col_idx)
    torch.cuda.synchronize()
    assert np.array_equal(oh.float().numpy(), res["out"])
    assert np.array_equal(fpl.row_ptr.cpu().numpy(), res["row_ptr"])


def _run(fp, fpl, q, k, v, gamma, tau, min_budget=0):
    import torch
    fpl.plan(q, k, tau)
    fpl.select(gamma, min_budget)
    out = torch.zeros_like(q)
    fpl.attn(q, k, v, out)
    dense = torch.zeros_like(q)
    fpl.dense(q, k, v, dense)
    torch.cuda.synchronize()
    return dict(pattern=fpl.pattern.cpu().numpy(), jsd=fpl.jsd.cpu().numpy(),
                row_ptr=fpl.row_ptr.cpu().numpy(), col_idx=fpl.col_idx.cpu().numpy(),
                out=out, dense=dense)


@pytest.mark.parametrize("n", [2048, 2085])
def test_token_major_batched_layout_bitwise(fp, n):
    """batch 2, [B][n][H][128] and [B][H][n][128] layouts vs two plain calls."""
    import torch
    H, G = 8, 2
    ws = [Workload(f"lay{b}", H, G, n, 0.9, 0.1, 0, 50 + b) for b in range(2)]
    bits = [gen.make_layer_bits(w) for w in ws]
    ref = []
    for w, (q, k, v) in zip(ws, bits):
        qt, kt, vt = (parity.to_torch_bf16(x) for x in (q, k, v))
        ref.append(_run(fp, fp.FlexPrefill(H, G, n), qt, kt, vt, 0.9, 0.1))
    # head-major batched: [B][H][n][d]
    qb, kb, vb = (torch.stack([parity.to_torch_bf16(b_[i]) for b_ in bits]) for i in range(3))
    got_h = _run(fp, fp.FlexPrefill(H, G, n, batch=2), qb, kb, vb, 0.9, 0.1)
    # token-major batched: [B][n][H][d] (a transposed copy of the same values)
    qs, ks, vs = (x.transpose(1, 2).contiguous() for x in (qb, kb, vb))
    got_s = _run(fp, fp.FlexPrefill(H, G, n, batch=2, layout="bshd"), qs, ks, vs, 0.9, 0.1)
    for got, to_bhsd in ((got_h, lambda x: x), (got_s, lambda x: x.transpose(1, 2))):
        for b in range(2):
            sl = slice(b * H, (b + 1) * H)
            for key in ("pattern", "jsd", "row_ptr"):
                assert np.array_equal(got[key][sl], ref[b][key]), (key, b)
            for h in range(H):  # the used part of each head's col_idx
                used = ref[b]["row_ptr"][h, -1]
                assert np.array_equal(got["col_idx"][b * H + h, :used], ref[b]["col_idx"][h, :used])
            assert torch.equal(to_bhsd(got["out"])[b], ref[b]["out"]), b
            assert torch.equal(to_bhsd(got["dense"])[b], ref[b]["dense"]), b


def test_token_major_output_rows_untouched_past_n(fp):
    """ragged n with token-major layout: rows >= n of a padded O buffer keep
    their contents (the kernel never writes past the sequence)."""
    import torch
    H, G, n = 4, 1, 1000
    w = Workload("pad", H, G, n, 0.9, 0.1, 0, 61)
    q, k, v = gen.make_layer_bits(w)
    qt, kt, vt = (parity.to_torch_bf16(x).transpose(0, 1).contiguous()[None] for x in (q, k, v))
    fpl = fp.FlexPrefill(H, G, n, layout="bshd")
    fpl.plan(qt, kt, 0.1)
    fpl.select(0.9, 0)
    big = torch.full((1, 1024, H, 128), 7.0, dtype=torch.bfloat16, device="cuda")
    fpl.attn(qt, kt, vt, big)  # O strides of an n-row tensor: rows 1000..1023 of `big` unused
    torch.cuda.synchronize()
    assert torch.all(big[0, n:] == 7.0)
    ref = parity.run_gpu(fp, w, q, k, v)["out"]
    assert np.array_equal(big[0, :n].transpose(0, 1).float().cpu().numpy(), ref)
