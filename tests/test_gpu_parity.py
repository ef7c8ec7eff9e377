"""GPU parity: the CUDA path through the C ABI vs the float64 oracle.

Tolerances (BASELINE.json north_star): pattern identical; selected sets
bit-exact except borderline elements (|C_{k-1} - gamma T| <= 1e-5 or a
near-tie of the threshold score), reported separately; outputs from bf16
with fp32 accumulation within max-abs 2e-2 and mean-abs 2e-3 of float64.
Stage-wise checks (oracle fed the GPU's inputs to that stage) use the
tighter bars of SURVEY.md §8(c) rule 1.
"""
import numpy as np
import pytest

import oracle
from synth import gen
from synth.configs import C1, Workload
from tests import parity

pytestmark = pytest.mark.gpu

MAX_ABS, MEAN_ABS = 2e-2, 2e-3


@pytest.fixture(scope="module")
def fp():
    import paper_2502_20766_b200 as m
    m.load_library()
    return m


def _oracle_plans(w, Q, K, heads=None, b=128):
    hs = range(w.heads) if heads is None else heads
    return {h: oracle.plan_head(Q[h], K[h * w.kv_heads // w.heads], b, w.tau) for h in hs}


def _check_plan(w, res, plans):
    dbg = res["dbg"]
    for h, p in plans.items():
        assert res["pattern"][h] == p["pattern"], (h, res["jsd"][h], p["D"])
        assert abs(res["jsd"][h] - p["D"]) <= 1e-4, (h, res["jsd"][h], p["D"])
        for key, dkey in (("a_v", "a_v"), ("a_s", "a_s"), ("a_hat", "a_hat"), ("a_bar", "a_bar")):
            rel, small = parity.rel_close(dbg[dkey][h], p[key], 1e-4, 1e-6)
            assert rel <= 1e-4 and small <= 1e-7, (h, key, rel, small)


def _check_select_stagewise(w, res, gamma, min_budget, b=128):
    dbg = res["dbg"]
    nb = -(-w.seq_len // b)
    for h in range(w.heads):
        pat = res["pattern"][h]
        cnt = dbg["sel_count"][h]
        if pat == oracle.VS:
            for seg, key in ((0, "a_v"), (1, "a_s")):
                x = dbg[key][h].astype(np.float64)
                sel = dbg["sel_v" if seg == 0 else "sel_s"][h, : cnt[seg]]
                assert np.all(np.diff(sel) > 0)
                mi, eo, bd, nbd = parity.classify(x, gamma, sel, parity.STAGE_DELTA, 0.0)
                assert mi == 0 and eo == 0 and bd == 0, (h, key, mi, eo, bd, nbd)
        else:
            tri = nb * (nb + 1) // 2
            x = dbg["A_bar"][h, :tri].astype(np.float64)
            sel = dbg["sel_qa"][h, : cnt[2]]
            assert np.all(np.diff(sel) > 0)
            mi, eo, bd, nbd = parity.classify(x, gamma, sel, parity.STAGE_DELTA, 0.0)
            assert mi == 0 and eo == 0 and bd == 0, (h, "A_bar", mi, eo, bd, nbd)
        # CSR bit-exact vs oracle O6-O9 on the GPU's sets and fp32 scores
        rp, ci = res["row_ptr"][h], res["col_idx"][h]
        assert parity.csr_rows_sorted(rp, ci, nb)
        M0, M = parity.stagewise_mask(pat, dbg, h, w.seq_len, gamma, min_budget, b)
        assert np.array_equal(parity.csr_mask(rp, ci, nb), M), h
        pre = oracle.add_forced(M0).sum(axis=1)
        assert np.array_equal(dbg["row_nnz_pre"][h], pre), h
        st = res["stats"][h]
        assert st["nnz_blocks"] == M.sum() and st["pattern"] == pat


def _check_attn_stagewise(w, res, Q, K, V, qblocks=None, b=128):
    nb = -(-w.seq_len // b)
    worst_max, worst_mean = 0.0, 0.0
    for h in range(w.heads):
        g = h * w.kv_heads // w.heads
        M = parity.csr_mask(res["row_ptr"][h], res["col_idx"][h], nb)
        ref = oracle.sparse_attention(Q[h], K[g], V[g], M, b, qblocks)
        rows = ~np.isnan(ref[:, 0])
        d = np.abs(res["out"][h][rows] - ref[rows])
        worst_max = max(worst_max, float(d.max()))
        worst_mean = max(worst_mean, float(d.mean()))
    assert worst_max <= MAX_ABS and worst_mean <= MEAN_ABS, (worst_max, worst_mean)
    return worst_max, worst_mean


def test_c1_full_parity(fp):
    res = full_parity(fp, C1)
    # both patterns trigger on the planted workload
    assert set(res["pattern"].tolist()) == {0, 1}


def full_parity(fp, w, b=128):
    """plan, stage-wise selection and attention, end-to-end sets (borderline
    rule) and outputs, and the dense kernel, all heads (block size b)."""
    q, k, v = gen.make_layer_bits(w)
    Q, K, V = parity.oracle_inputs(q, k, v)
    res = parity.run_gpu(fp, w, q, k, v, dense=True, block_size=b)
    plans = _oracle_plans(w, Q, K, b=b)
    _check_plan(w, res, plans)
    _check_select_stagewise(w, res, w.gamma, w.min_budget, b)
    _check_attn_stagewise(w, res, Q, K, V, b=b)
    # end-to-end: oracle from scratch, borderline rule
    nb = -(-w.seq_len // b)
    for h in range(w.heads):
        g = h * w.kv_heads // w.heads
        o = oracle.flexprefill_head(Q[h], K[g], V[g], b, w.gamma, w.tau, w.min_budget,
                                    with_output=False)
        cnt = res["dbg"]["sel_count"][h]
        if o["pattern"] == oracle.VS:
            for seg, key in ((0, "a_v"), (1, "a_s")):
                sel = res["dbg"]["sel_v" if seg == 0 else "sel_s"][h, : cnt[seg]]
                mi, eo, bd, nbd = parity.classify(o[key], w.gamma, sel)
                assert mi == 0 and eo == 0, (h, key, mi, eo)
        else:
            vals, _, _ = oracle.qa_flat(o["Abar"])
            mi, eo, bd, nbd = parity.classify(vals, w.gamma, res["dbg"]["sel_qa"][h, : cnt[2]])
            assert mi == 0 and eo == 0, (h, mi, eo)
        # rows whose block lists match: outputs vs oracle output on the oracle's set
        Mg = parity.csr_mask(res["row_ptr"][h], res["col_idx"][h], nb)
        same = np.all(Mg == o["mask"], axis=1)
        ref = oracle.sparse_attention(Q[h], K[g], V[g], o["mask"], b, np.nonzero(same)[0])
        rows = ~np.isnan(ref[:, 0])
        if rows.any():
            d = np.abs(res["out"][h][rows] - ref[rows])
            assert d.max() <= MAX_ABS and d.mean() <= MEAN_ABS
    # dense kernel vs oracle dense causal attention
    for h in range(w.heads):
        g = h * w.kv_heads // w.heads
        ref = oracle.dense_causal_attention(Q[h], K[g], V[g])
        d = np.abs(res["dense"][h] - ref)
        assert d.max() <= MAX_ABS and d.mean() <= MEAN_ABS, (h, d.max(), d.mean())
    return res


def test_gamma_one_equals_dense(fp):
    w = C1.with_(gamma=1.0)
    q, k, v = gen.make_layer_bits(w)
    res = parity.run_gpu(fp, w, q, k, v, gamma=1.0, dense=True)
    nb = -(-w.seq_len // 128)
    for h in range(w.heads):
        assert res["row_ptr"][h][-1] == nb * (nb + 1) // 2
    # same kernel, same block order -> bitwise identical to the dense kernel
    assert np.array_equal(res["out"], res["dense"])


def test_ragged_chunks_gqa_and_min_budget(fp):
    # n = 4224: 33 blocks -> the last representative chunk holds one tile; g = 4
    w = Workload("ragged", 8, 2, 4224, 0.9, 0.1, 1024, 7)
    q, k, v = gen.make_layer_bits(w)
    Q, K, V = parity.oracle_inputs(q, k, v)
    res = parity.run_gpu(fp, w, q, k, v)
    _check_plan(w, res, _oracle_plans(w, Q, K))
    _check_select_stagewise(w, res, w.gamma, w.min_budget)
    assert sum(s["budget_added"] for s in res["stats"]) > 0
    _check_attn_stagewise(w, res, Q, K, V)


@pytest.mark.parametrize("gamma", [0.8, 0.95, 0.99])
def test_glm_layout_gamma_sweep(fp, gamma):
    # GLM-like group size 16 (32 Q / 2 KV), reduced length
    w = Workload("glm-small", 32, 2, 2048, gamma, 0.1, 1024, 104)
    q, k, v = gen.make_layer_bits(w)
    Q, K, V = parity.oracle_inputs(q, k, v)
    res = parity.run_gpu(fp, w, q, k, v, gamma=gamma)
    _check_plan(w, res, _oracle_plans(w, Q, K, heads=[0, 1, 15, 16, 31]))
    _check_select_stagewise(w, res, gamma, w.min_budget)
    _check_attn_stagewise(w, res, Q, K, V, qblocks=[0, 1, 7, 15])


@pytest.mark.parametrize("n", [128, 256])
def test_tiny_sequences(fp, n):
    w = Workload("tiny", 4, 2, n, 0.9, 0.1, 0, 11)
    q, k, v = gen.make_layer_bits(w)
    Q, K, V = parity.oracle_inputs(q, k, v)
    res = parity.run_gpu(fp, w, q, k, v, dense=True)
    _check_plan(w, res, _oracle_plans(w, Q, K))
    _check_select_stagewise(w, res, w.gamma, 0)
    _check_attn_stagewise(w, res, Q, K, V)


def test_ragged_chunk_multi_tile(fp):
    # 65 blocks, 32 heads: 4-tile representative chunks with a 1-tile last chunk
    w = Workload("ragged-ct4", 32, 8, 8320, 0.9, 0.1, 0, 9)
    q, k, v = gen.make_layer_bits(w)
    Q, K, V = parity.oracle_inputs(q, k, v)
    res = parity.run_gpu(fp, w, q, k, v)
    _check_plan(w, res, _oracle_plans(w, Q, K, heads=[0, 3, 17, 30]))
    _check_select_stagewise(w, res, w.gamma, 0)


def test_cuda_graph_replay_matches_eager(fp):
    import torch
    w = Workload("graph", 8, 2, 4096, 0.9, 0.1, 0, 13)
    q, k, v = gen.make_layer_bits(w)
    eager = parity.run_gpu(fp, w, q, k, v)
    qt, kt, vt = (parity.to_torch_bf16(x) for x in (q, k, v))
    fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
    out = torch.zeros_like(qt)
    graph = fpl.capture_layer(qt, kt, vt, out, w.gamma, w.tau, 0)
    out.zero_()
    graph.replay()
    torch.cuda.synchronize()
    assert np.array_equal(out.float().cpu().numpy(), eager["out"])


def test_determinism(fp):
    w = Workload("det", 8, 2, 4096, 0.9, 0.1, 0, 5)
    q, k, v = gen.make_layer_bits(w)
    r1 = parity.run_gpu(fp, w, q, k, v)
    r2 = parity.run_gpu(fp, w, q, k, v)
    for key in ("pattern", "jsd", "row_ptr", "col_idx", "out"):
        assert np.array_equal(r1[key], r2[key]), key
    for key in ("a_v", "a_s", "A_bar", "sel_v", "sel_s", "sel_qa"):
        assert np.array_equal(r1["dbg"][key], r2["dbg"][key]), key


def test_abi_errors_enqueue_nothing(fp):
    import torch
    w = Workload("err", 4, 1, 1024, 0.9, 0.1, 0, 3)
    fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
    q = torch.zeros(4, 1024, 128, dtype=torch.bfloat16, device="cuda")
    k = torch.zeros(1, 1024, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(fp.FlexPrefillError) as e:
        fp.fp_plan(q, k, 4, 1, 1024, 1.5, fpl.ws, fpl.ws_bytes, fpl.pattern, fpl.jsd)
    assert e.value.status == 3
    with pytest.raises(fp.FlexPrefillError) as e:
        fp.fp_plan(q, k, 4, 1, 1024, 0.1, fpl.ws, 16, fpl.pattern, fpl.jsd)
    assert e.value.status == 5
    with pytest.raises(fp.FlexPrefillError) as e:
        fp.fp_plan(q.data_ptr() + 2, k, 4, 1, 1024, 0.1, fpl.ws, fpl.ws_bytes, fpl.pattern, fpl.jsd)
    assert e.value.status == 4
    with pytest.raises(fp.FlexPrefillError) as e:
        fp.fp_select(4, 1, 1024, 0.0, 0, fpl.ws, fpl.ws_bytes, fpl.row_ptr, fpl.col_idx)
    assert e.value.status == 3
    torch.cuda.synchronize()


def test_layer_host_e2e_matches_device_path(fp):
    import torch
    w = C1
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


def test_tau_sweep_mixed_heads(fp):
    # C5-style mixed heads spread D across the swept taus; the decision flips per tau
    from synth.configs import C5_QWEN, C5_TAUS
    w = C5_QWEN.with_(seq_len=4096)
    q, k, v = gen.make_layer_bits(w)
    Q, K, V = parity.oracle_inputs(q, k, v)
    plans = _oracle_plans(w, Q, K)
    flips = set()
    for tau in C5_TAUS:
        res = parity.run_gpu(fp, w.with_(tau=tau), q, k, v, want_out=False)
        for h, p in plans.items():
            assert abs(res["jsd"][h] - p["D"]) <= 1e-4, (tau, h)
            assert res["pattern"][h] == (1 if p["D"] < tau else 0), (tau, h, p["D"])
        flips.add(int(res["pattern"].sum()))
    assert len(flips) >= 3  # the number of QA heads changes across the sweep


@pytest.mark.parametrize("vs_mode,qa_mode,min_budget,max_budget",
                         [(1, 0, 0, 0), (0, 1, 0, 0), (1, 1, 1024, 0), (0, 0, 0, 1024),
                          (1, 1, 512, 768)])
def test_selection_variants_stagewise(fp, vs_mode, qa_mode, min_budget, max_budget):
    """f1 (block-pooled VS lines), f2 (per-row QA selection, maximum budget):
    stage-wise parity of the sets and the CSR, attention on the result."""
    w = Workload("variants", 8, 2, 4096, 0.9, 0.1, min_budget, 17)
    q, k, v = gen.make_layer_bits(w)
    Q, K, V = parity.oracle_inputs(q, k, v)
    res = parity.run_gpu(fp, w, q, k, v, vs_mode=vs_mode, qa_mode=qa_mode, max_budget=max_budget)
    dbg = res["dbg"]
    nb = -(-w.seq_len // 128)
    assert set(res["pattern"].tolist()) == {0, 1}
    for h in range(w.heads):
        pat = res["pattern"][h]
        cnt = dbg["sel_count"][h]
        if pat == oracle.VS:
            if vs_mode == 1:
                segs = ((dbg["a_hat"][h], dbg["sel_v"][h, : cnt[0]]),
                        (dbg["As"][h], dbg["sel_s"][h, : cnt[1]]))
            else:
                segs = ((dbg["a_v"][h], dbg["sel_v"][h, : cnt[0]]),
                        (dbg["a_s"][h], dbg["sel_s"][h, : cnt[1]]))
            for x, sel in segs:
                mi, eo, bd, _ = parity.classify(x.astype(np.float64), w.gamma, sel, parity.STAGE_DELTA, 0.0)
                assert mi == 0 and eo == 0 and bd == 0, (h, vs_mode)
        M0, M = parity.stagewise_mask(pat, dbg, h, w.seq_len, w.gamma, min_budget, vs_mode=vs_mode,
                                      qa_mode=qa_mode, max_budget=max_budget)
        rp, ci = res["row_ptr"][h], res["col_idx"][h]
        assert parity.csr_rows_sorted(rp, ci, nb)
        assert np.array_equal(parity.csr_mask(rp, ci, nb), M), (h, vs_mode, qa_mode)
        if max_budget:
            m = -(-max_budget // 128)
            assert np.all(np.diff(rp) <= np.maximum(m, 2))
    if max_budget:
        assert sum(s["budget_removed"] for s in res["stats"]) > 0
    _check_attn_stagewise(w, res, Q, K, V, qblocks=[0, 1, 15, 31])
