"""Next row f3: block_size = 64 (the paper's Triton block
size ablation). The whole path runs with 64-token blocks: Q^ is the
last 64 query rows, pooled estimates and line rasterisation use
64-blocks, and the attention computes exactly the selected 64 x 64 blocks
(fp_attn8.cu: coarse 128 x 128 tensor-core tiles with per-quadrant masks).
Parity against the float64 oracle run with b = 64."""
import numpy as np
import pytest

import oracle
from synth import gen
from synth.configs import Workload
from tests import parity
from tests.test_gpu_parity import (MAX_ABS, MEAN_ABS, _check_attn_stagewise, _check_plan,
                                   _check_select_stagewise, _oracle_plans, full_parity)

pytestmark = pytest.mark.gpu
B = 64


@pytest.fixture(scope="module")
def fp():
    import paper_2502_20766_b200 as m
    m.load_library()
    return m


@pytest.mark.parametrize("heads,kv,n,gamma,min_budget", [
    (4, 1, 2048, 0.9, 0),        # C1 layout: 32 blocks of 64
    (8, 2, 2085, 0.95, 1024),    # ragged: last 64-block holds 37 rows; min budget 16 blocks
    (4, 2, 1000, 0.9, 0),        # 16 blocks (last 40 rows): the last coarse tile has no row B
    (4, 1, 128, 0.9, 0),         # two blocks, one coarse tile
])
def test_block64_full_parity(fp, heads, kv, n, gamma, min_budget):
    w = Workload(f"b64-{n}", heads, kv, n, gamma, 0.1, min_budget, 90 + n % 89)
    res = full_parity(fp, w, b=B)
    nb = -(-n // B)
    assert res["row_ptr"].shape[1] == nb + 1
    assert all(s_["nnz_blocks"] >= 2 * nb - 1 for s_ in res["stats"])  # forced blocks


def test_block64_both_patterns_and_finer_sets(fp):
    """the C1 workload selects both patterns at b = 64 too, and the 64-block
    sets are no coarser than the 128-block ones (each selected 128-block of
    the b = 128 run is covered by the b = 64 selection's 64-blocks at >= 1/4)."""
    w = Workload("b64-c1", 4, 1, 2048, 0.9, 0.1, 0, 101)
    q, k, v = gen.make_layer_bits(w)
    r64 = parity.run_gpu(fp, w, q, k, v, block_size=64)
    assert set(r64["pattern"].tolist()) == {0, 1}
    nb = 32
    for h in range(w.heads):
        M = parity.csr_mask(r64["row_ptr"][h], r64["col_idx"][h], nb)
        assert parity.csr_rows_sorted(r64["row_ptr"][h], r64["col_idx"][h], nb)
        assert M.sum() < nb * (nb + 1) // 2  # sparse


@pytest.mark.parametrize("n,density,seed", [(2048, 0.3, 1), (2085, 0.5, 2), (4096, 0.15, 3)])
def test_block64_attention_random_masks(fp, n, density, seed):
    """fp_sparse_attn on random 64-block CSRs (each row: block 0, its diagonal,
    random others): every quadrant combination of the coarse tiles, ragged n."""
    import torch
    H, G = 4, 2
    w = Workload(f"b64-rand-{n}", H, G, n, 0.9, 0.1, 0, 120 + seed)
    q, k, v = gen.make_layer_bits(w)
    Q, K, V = parity.oracle_inputs(q, k, v)
    nb = -(-n // B)
    rng = np.random.default_rng(seed)
    masks, rp, ci = [], [], []
    cap = nb * (nb + 1) // 2
    for h in range(H):
        M = np.tril(rng.random((nb, nb)) < density)
        M[:, 0] = True
        M[np.arange(nb), np.arange(nb)] = True
        masks.append(M)
        r = np.zeros(nb + 1, np.int32)
        c = np.zeros(cap, np.int32)
        off = 0
        for qb in range(nb):
            ks = np.nonzero(M[qb, : qb + 1])[0]
            c[off: off + len(ks)] = ks
            off += len(ks)
            r[qb + 1] = off
        rp.append(r)
        ci.append(c)
    qt, kt, vt = (parity.to_torch_bf16(x) for x in (q, k, v))
    rpt = torch.from_numpy(np.stack(rp)).cuda()
    cit = torch.from_numpy(np.stack(ci)).cuda()
    out = torch.zeros_like(qt)
    fp.fp_sparse_attn(qt, kt, vt, out, H, G, n, rpt, cit, block_size=B)
    torch.cuda.synchronize()
    got = out.float().cpu().numpy()
    for h in range(H):
        ref = oracle.sparse_attention(Q[h], K[h * G // H], V[h * G // H], masks[h], B)
        d = np.abs(got[h] - ref)
        assert d.max() <= MAX_ABS and d.mean() <= MEAN_ABS, (h, d.max(), d.mean())


def test_block64_gamma_one_is_dense(fp):
    """gamma >= 1 selects every causal 64-block: the output is dense causal
    attention (oracle), and the layer's dense kernel agrees."""
    w = Workload("b64-g1", 4, 1, 1000, 1.0, 0.1, 0, 131)
    q, k, v = gen.make_layer_bits(w)
    Q, K, V = parity.oracle_inputs(q, k, v)
    res = parity.run_gpu(fp, w, q, k, v, gamma=1.0, dense=True, block_size=B)
    nb = -(-1000 // B)
    assert np.all(res["row_ptr"][:, -1] == nb * (nb + 1) // 2)
    for h in range(w.heads):
        ref = oracle.dense_causal_attention(Q[h], K[0], V[0])
        for key in ("out", "dense"):
            d = np.abs(res[key][h] - ref)
            assert d.max() <= MAX_ABS and d.mean() <= MEAN_ABS, (key, h, d.max())


def test_block64_glm_group16_stagewise(fp):
    """GQA group 16 (GLM-like) at b = 64 with min budget: plan, selection and
    attention stage-wise on a subset of heads / q-blocks."""
    w = Workload("b64-glm", 32, 2, 2048, 0.95, 0.1, 1024, 104)
    q, k, v = gen.make_layer_bits(w)
    Q, K, V = parity.oracle_inputs(q, k, v)
    res = parity.run_gpu(fp, w, q, k, v, block_size=B)
    _check_plan(w, res, _oracle_plans(w, Q, K, heads=[0, 1, 15, 16, 31], b=B))
    _check_select_stagewise(w, res, w.gamma, w.min_budget, B)
    _check_attn_stagewise(w, res, Q, K, V, qblocks=[0, 1, 7, 15, 16, 31], b=B)


def test_block64_layer_host_matches_device_path(fp):
    """the host-buffer pipeline (fp_layer_host) at b = 64 gives the device path's
    CSR and outputs bitwise."""
    import torch
    w = Workload("b64-host", 8, 2, 2085, 0.9, 0.1, 512, 141)
    q, k, v = gen.make_layer_bits(w)
    res = parity.run_gpu(fp, w, q, k, v, block_size=B)
    fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len, block_size=B)
    qh, kh, vh = (torch.from_numpy(x).view(torch.bfloat16).pin_memory() for x in (q, k, v))
    oh = torch.empty_like(qh).pin_memory()
    dq, dk, dv = (torch.empty(x.shape, dtype=torch.bfloat16, device="cuda") for x in (qh, kh, vh))
    do = torch.empty_like(dq)
    fp.fp_layer_host(qh, kh, vh, oh, dq, dk, dv, do, w.heads, w.kv_heads, w.seq_len, w.gamma, w.tau,
                     w.min_budget, fpl.ws, fpl.ws_bytes, fpl.pattern, fpl.jsd, fpl.row_ptr,
                     fpl.col_idx, block_size=B)
    torch.cuda.synchronize()
    assert np.array_equal(fpl.row_ptr.cpu().numpy(), res["row_ptr"])
    assert np.array_equal(oh.float().numpy(), res["out"])


def test_block64_peers(fp):
    """b = 64 runs the same (v8) attention kernel on coarse tiles, so the fused
    output exchange works there too: every peer buffer receives exactly the
    plain call's rows, bitwise."""
    import torch
    w = Workload("b64-peers", 4, 1, 1024, 0.9, 0.1, 0, 143)
    q, k, v = (parity.to_torch_bf16(x) for x in gen.make_layer_bits(w))
    fpl = fp.FlexPrefill(4, 1, 1024, block_size=B)
    fpl.plan(q, k, 0.1)
    fpl.select(0.9, 0)
    ref = torch.zeros_like(q)
    fpl.attn(q, k, v, ref)
    out = torch.zeros_like(q)
    peer = torch.zeros_like(q)
    ptrs = torch.tensor([peer.data_ptr()], dtype=torch.int64, device="cuda")
    fp.fp_sparse_attn_peers(q, k, v, out, ptrs, 1, 4, 1, 1024, fpl.row_ptr, fpl.col_idx,
                            ws=fpl.ws, ws_bytes=fpl.ws_bytes, block_size=B)
    torch.cuda.synchronize()
    assert torch.equal(out, ref) and torch.equal(peer, ref)


@pytest.mark.slow
def test_block64_32k_sampled(fp):
    """b = 64 at full size (Llama-like 32/8 at 32k, the coarse-tile path of the
    v8 kernel): end-to-end parity on sampled heads of both patterns and sampled
    64-row query blocks against the b = 64 oracle (pattern, sets with borderline
    elements reported, outputs within the north-star tolerance)."""
    from synth.configs import C2
    w = C2
    q, k, v = gen.make_layer_bits(w)
    res = parity.run_gpu(fp, w, q, k, v, block_size=B)
    nb = -(-w.seq_len // B)
    for h in range(w.heads):  # whole-layer CSR properties: sorted rows, forced blocks
        rp, ci = res["row_ptr"][h], res["col_idx"][h]
        assert rp[0] == 0 and np.all(np.diff(rp) >= np.minimum(np.arange(nb) + 1, 2))
    heads = [0, 3]  # a Vertical-Slash-type and a Query-Aware-type head (synth/gen.py)
    qbs = sorted({0, 1, 2, 3, nb // 2, nb // 2 + 1, nb - 2, nb - 1})
    pats = set()
    for h in heads:
        g = h * w.kv_heads // w.heads
        rep = parity.head_report(w, h, res, gen.bits_to_f64(q[h]), gen.bits_to_f64(k[g]),
                                 gen.bits_to_f64(v[g]), qbs, b=B)
        parity.check_report(rep)
        pats.add(rep["pattern_oracle"])
    assert pats == {0, 1}
