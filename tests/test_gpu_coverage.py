"""GPU parity on every configuration the bench reports (VERDICT r01 "next" #1):
the Yi-9B-like 32/4 layout at 32k and 128k, the C5 mixed-head tau sweep at
32k, the GLM-like C4 gamma sweep ends (0.8, 0.99) at 128k with the minimum
budget on, and the f1 / f2 selection variants at 32k.

Each case runs the whole layer through the binding in the launch
configuration bench.py times, then, on sampled heads (both patterns) and
sampled q-blocks (always 0, 1, nb/2, nb-1):
  * stage-wise: top-mass sets bit-exact against the oracle's topmass on the
    GPU's own fp32 scores, CSR bit-exact against O6-O9 on the GPU's sets;
  * end-to-end (oracle from scratch on the same bf16 inputs,
    parity.head_report): pattern identical, |dD| <= 1e-4, a_v/a_s/a_hat/a_bar
    within 1e-4 relative, K_bar / Q_bar / A_bar values, every "in" element
    selected and no "out" element, borderline differences reported
    (north_star: "reported separately"), outputs within max-abs 2e-2 /
    mean-abs 2e-3 on the GPU's CSR and, on rows whose lists match, on the
    oracle's own mask.
The reports are printed in pytest's terminal summary (tests/conftest.py).
"""
import numpy as np
import pytest

import oracle
from synth import gen
from synth.configs import C2, C4, C5_QWEN, C5_TAUS, C5_YI
from tests import parity

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def fp():
    import paper_2502_20766_b200 as m
    m.load_library()
    return m


def _sample_heads(w, k):
    """k heads: half VS-type, half QA-type by construction (synth/gen.py)."""
    vs = [h for h in range(w.heads) if not gen.is_qa_type(h, w.heads, w.kv_heads)]
    qa = [h for h in range(w.heads) if gen.is_qa_type(h, w.heads, w.kv_heads)]
    rng = np.random.default_rng(w.seed + w.seq_len)
    pick = list(rng.choice(vs, k - k // 2, replace=False)) + list(rng.choice(qa, k // 2, replace=False))
    return sorted(int(h) for h in pick)


def _qblocks(nb, seed=7):
    rng = np.random.default_rng(seed)
    return sorted({0, 1, nb // 2, nb - 1, *rng.integers(0, nb, 3).tolist()})


def _stagewise(w, res, heads, gamma, min_budget, vs_mode=0, qa_mode=0, max_budget=0):
    dbg = res["dbg"]
    nb = -(-w.seq_len // 128)
    for h in heads:
        pat = res["pattern"][h]
        cnt = dbg["sel_count"][h]
        if pat == oracle.VS:
            if vs_mode == 1:
                segs = ((dbg["a_hat"][h], dbg["sel_v"][h, : cnt[0]]), (dbg["As"][h], dbg["sel_s"][h, : cnt[1]]))
            else:
                segs = ((dbg["a_v"][h], dbg["sel_v"][h, : cnt[0]]), (dbg["a_s"][h], dbg["sel_s"][h, : cnt[1]]))
        elif qa_mode == 0:
            segs = ((dbg["A_bar"][h, : nb * (nb + 1) // 2], dbg["sel_qa"][h, : cnt[2]]),)
        else:
            segs = ()
        for x, sel in segs:
            assert np.all(np.diff(sel) > 0), h
            mi, eo, bd, _ = parity.classify(x.astype(np.float64), gamma, sel, parity.STAGE_DELTA, 0.0)
            assert mi == 0 and eo == 0 and bd == 0, (h, mi, eo, bd)
        rp, ci = res["row_ptr"][h], res["col_idx"][h]
        assert parity.csr_rows_sorted(rp, ci, nb), h
        _, M = parity.stagewise_mask(pat, dbg, h, w.seq_len, gamma, min_budget, vs_mode=vs_mode,
                                     qa_mode=qa_mode, max_budget=max_budget)
        assert np.array_equal(parity.csr_mask(rp, ci, nb), M), h


def _case(fp, w, k_heads, gamma=None, tau=None, min_budget=None, vs_mode=0, qa_mode=0,
          max_budget=0, bits=None):
    gamma = w.gamma if gamma is None else gamma
    tau = w.tau if tau is None else tau
    min_budget = w.min_budget if min_budget is None else min_budget
    q, k, v = gen.make_layer_bits(w) if bits is None else bits
    res = parity.run_gpu(fp, w, q, k, v, gamma=gamma, tau=tau, min_budget=min_budget,
                         vs_mode=vs_mode, qa_mode=qa_mode, max_budget=max_budget)
    nb = -(-w.seq_len // 128)
    m = -(-min_budget // 128) if min_budget else 0
    for h in range(w.heads):  # whole-layer properties, every head
        rp, ci = res["row_ptr"][h], res["col_idx"][h]
        assert rp[0] == 0 and np.all(np.diff(rp) >= np.minimum(np.arange(nb) + 1, max(m, 1))), h
    heads = _sample_heads(w, k_heads)
    _stagewise(w, res, heads, gamma, min_budget, vs_mode, qa_mode, max_budget)
    qbs = _qblocks(nb)
    reps = []
    for h in heads:
        g = h * w.kv_heads // w.heads
        rep = parity.head_report(w, h, res, gen.bits_to_f64(q[h]), gen.bits_to_f64(k[g]),
                                 gen.bits_to_f64(v[g]), qbs, gamma=gamma, tau=tau,
                                 min_budget=min_budget, vs_mode=vs_mode, qa_mode=qa_mode,
                                 max_budget=max_budget)
        parity.check_report(rep)
        reps.append(rep)
    return res, reps


def test_yi_32_4_32k(fp):
    w = C5_YI.with_(seq_len=32768)
    res, reps = _case(fp, w, 4)
    assert {r["pattern_oracle"] for r in reps} == {0, 1}


def test_yi_32_4_128k(fp):
    w = C5_YI.with_(seq_len=131072)
    _case(fp, w, 2)


def test_qwen_28_4_128k(fp):
    w = C5_QWEN.with_(seq_len=131072)
    _case(fp, w, 2)


@pytest.mark.parametrize("base", [C5_QWEN, C5_YI], ids=["qwen28_4", "yi32_4"])
def test_c5_mixed_heads_32k_tau_sweep(fp, base):
    """Mixed heads spread D over the swept taus (synth/gen.py): every head's D
    and pattern at every tau against the oracle, end-to-end reports at the
    sweep ends."""
    w = base.with_(seq_len=32768)
    bits = gen.make_layer_bits(w)
    q, k, _ = bits
    D = np.array([oracle.plan_head(gen.bits_to_f64(q[h]), gen.bits_to_f64(k[h * w.kv_heads // w.heads]),
                                   128, 0.1)["D"] for h in range(w.heads)])
    counts = set()
    for tau in C5_TAUS:
        res = parity.run_gpu(fp, w, *bits, tau=tau, want_out=False)
        assert np.abs(res["jsd"] - D).max() <= 1e-4
        near = np.abs(D - tau) < 1e-4
        want = (D < tau).astype(np.int32)
        assert np.array_equal(res["pattern"][~near], want[~near]), tau
        counts.add(int(res["pattern"].sum()))
    assert len(counts) >= 2  # the number of QA heads changes across the sweep
    for tau in (C5_TAUS[0], C5_TAUS[-1]):
        _case(fp, w.with_(tau=tau), 2, bits=bits)


@pytest.mark.parametrize("gamma", [0.8, 0.99])
def test_c4_glm_128k_gamma_ends_min_budget(fp, gamma):
    res, _ = _case(fp, C4.with_(gamma=gamma), 2)
    if gamma == 0.8:  # at low gamma the floor binds on sparse rows
        assert sum(s["budget_added"] for s in res["stats"]) > 0


@pytest.mark.parametrize("vs_mode,qa_mode,min_budget,max_budget",
                         [(1, 0, 0, 0), (0, 1, 0, 0), (1, 1, 1024, 0), (0, 0, 1024, 4096)],
                         ids=["f1", "f2rows", "f1f2min", "minmax"])
def test_selection_variants_32k(fp, vs_mode, qa_mode, min_budget, max_budget):
    res, _ = _case(fp, C2, 2, min_budget=min_budget, vs_mode=vs_mode, qa_mode=qa_mode,
                   max_budget=max_budget)
    if max_budget:
        m = -(-max_budget // 128)
        assert np.all(np.diff(res["row_ptr"], axis=1) <= m)
        assert sum(s["budget_removed"] for s in res["stats"]) > 0


def test_layer_host_and_head_slices_bitwise_32k(fp):
    """The host-buffer pipeline (one head at a time for the first KV group, then
    whole groups) and single-head / single-group calls give bitwise the
    whole-layer device result at 32k (the representative-pass chunking depends
    on n only)."""
    import torch
    w = C2
    q, k, v = gen.make_layer_bits(w)
    res = parity.run_gpu(fp, w, q, k, v)
    fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
    qh, kh, vh = (torch.from_numpy(x).view(torch.bfloat16).pin_memory() for x in (q, k, v))
    oh = torch.empty_like(qh).pin_memory()
    dq, dk, dv = (torch.empty(x.shape, dtype=torch.bfloat16, device="cuda") for x in (qh, kh, vh))
    do = torch.empty_like(dq)
    fp.fp_layer_host(qh, kh, vh, oh, dq, dk, dv, do, w.heads, w.kv_heads, w.seq_len, w.gamma, w.tau,
                     w.min_budget, fpl.ws, fpl.ws_bytes, fpl.pattern, fpl.jsd, fpl.row_ptr, fpl.col_idx)
    torch.cuda.synchronize()
    assert np.array_equal(oh.float().numpy(), res["out"])
    assert np.array_equal(fpl.pattern.cpu().numpy(), res["pattern"])
    assert np.array_equal(fpl.jsd.cpu().numpy(), res["jsd"])
    assert np.array_equal(fpl.row_ptr.cpu().numpy(), res["row_ptr"])
    # one head alone and one KV group alone: plan values bitwise equal
    g = w.heads // w.kv_heads
    for h0, nh, kv0, nkv in ((5, 1, 1, 1), (8, g, 2, 1)):
        f1 = fp.FlexPrefill(nh, nkv, w.seq_len)
        qt = torch.from_numpy(q[h0:h0 + nh]).view(torch.bfloat16).cuda()
        kt = torch.from_numpy(k[kv0:kv0 + nkv]).view(torch.bfloat16).cuda()
        f1.plan(qt, kt, w.tau)
        f1.select(w.gamma, w.min_budget)
        torch.cuda.synchronize()
        d1 = f1.debug()
        for key in ("a_v", "a_s", "a_hat", "a_bar"):
            assert np.array_equal(d1[key].numpy(), res["dbg"][key][h0:h0 + nh]), (h0, key)
        assert np.array_equal(f1.jsd.cpu().numpy(), res["jsd"][h0:h0 + nh])
        assert np.array_equal(f1.row_ptr.cpu().numpy(), res["row_ptr"][h0:h0 + nh])


def test_layer_host_invalid_call_enqueues_nothing(fp):
    """A validation error of fp_layer_host is returned before the first copy:
    the device buffers keep their sentinel contents."""
    import torch
    H, G, n = 8, 2, 2048
    fpl = fp.FlexPrefill(H, G, n)
    qh = torch.ones(H, n, 128, dtype=torch.bfloat16).pin_memory()
    kh = torch.ones(G, n, 128, dtype=torch.bfloat16).pin_memory()
    oh = torch.zeros_like(qh).pin_memory()
    dq = torch.full((H, n, 128), 7.0, dtype=torch.bfloat16, device="cuda")
    dk = torch.full((G, n, 128), 7.0, dtype=torch.bfloat16, device="cuda")
    dv = dk.clone()
    do = dq.clone()
    torch.cuda.synchronize()
    bad_rp = fpl.row_ptr.data_ptr() + 2  # misaligned int32 array, the last check
    with pytest.raises(fp.FlexPrefillError) as e:
        fp.fp_layer_host(qh, kh, kh, oh, dq, dk, dv, do, H, G, n, 0.9, 0.1, 0, fpl.ws, fpl.ws_bytes,
                         fpl.pattern, fpl.jsd, bad_rp, fpl.col_idx)
    assert e.value.status == 4
    torch.cuda.synchronize()
    assert bool((dq == 7.0).all()) and bool((dk == 7.0).all()) and bool((do == 7.0).all())
    assert bool((oh == 0).all())


def test_head_slices_csr_bitwise_64k(fp):
    """The top-mass cluster size depends on how many heads a call batches (more
    CTAs per head while the grid fits one wave: C = 4 for the 32-head layer, 8
    for one head or one KV group at 64k); the selection is exact integer
    arithmetic over the same scores, so the CSR (row_ptr AND col_idx) of a head
    must not depend on it (head-partitioned multi-GPU runs rely on this)."""
    import torch
    w = C2.with_(seq_len=65536)
    q, k, _ = gen.make_layer_bits(w)
    full = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
    qa = torch.from_numpy(q).view(torch.bfloat16).cuda()
    ka = torch.from_numpy(k).view(torch.bfloat16).cuda()
    full.plan(qa, ka, w.tau)
    full.select(w.gamma, w.min_budget)
    torch.cuda.synchronize()
    rp_all, ci_all = full.row_ptr.cpu().numpy(), full.col_idx.cpu().numpy()
    g = w.heads // w.kv_heads
    for h0, nh, kv0, nkv in ((3, 1, 0, 1), (12, g, 3, 1)):
        f1 = fp.FlexPrefill(nh, nkv, w.seq_len)
        qt = torch.from_numpy(q[h0:h0 + nh]).view(torch.bfloat16).cuda()
        kt = torch.from_numpy(k[kv0:kv0 + nkv]).view(torch.bfloat16).cuda()
        f1.plan(qt, kt, w.tau)
        f1.select(w.gamma, w.min_budget)
        torch.cuda.synchronize()
        rp, ci = f1.row_ptr.cpu().numpy(), f1.col_idx.cpu().numpy()
        assert np.array_equal(rp, rp_all[h0:h0 + nh]), (h0, nh)
        for j in range(nh):
            nnz = int(rp[j, -1])
            assert np.array_equal(ci[j, :nnz], ci_all[h0 + j, :nnz]), (h0 + j)
