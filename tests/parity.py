"""Parity checker: CUDA path (through the C ABI) vs the float64 oracle.

Test infrastructure (may import oracle/). Implements SURVEY.md §8(c) "Parity
rules": stage-wise checks (the oracle fed the GPU's own inputs to a stage)
and the end-to-end borderline classifier with delta = 1e-5 (north_star:
"bit-exact, except for blocks whose fp32 scores lie within 1e-5 of the
cumulative threshold, which are reported separately").
"""
import numpy as np

import oracle

REPORTS = []  # head_report dicts of this session (printed by conftest's terminal summary)

DELTA = 1e-5        # end-to-end borderline window on C_{k-1} - gamma T
STAGE_DELTA = 1e-12  # stage-wise: summation-order ties only
LAM_REL = 1e-5      # near-tie window around the K-th score (Appendix B lambda)


def to_torch_bf16(bits, device="cuda"):
    import torch
    return torch.from_numpy(np.ascontiguousarray(bits)).view(torch.bfloat16).to(device)


def run_gpu(fp, w, q_bits, k_bits, v_bits, gamma=None, tau=None, min_budget=None, dense=False,
            want_out=True, vs_mode=0, qa_mode=0, max_budget=0, block_size=128):
    """Run plan -> select -> attn through the binding; return host copies."""
    import torch
    gamma = w.gamma if gamma is None else gamma
    tau = w.tau if tau is None else tau
    min_budget = w.min_budget if min_budget is None else min_budget
    q, k, v = (to_torch_bf16(x) for x in (q_bits, k_bits, v_bits))
    fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len, block_size=block_size)
    fpl.plan(q, k, tau)
    fpl.select(gamma, min_budget, vs_mode=vs_mode, qa_mode=qa_mode, max_budget=max_budget)
    out = torch.empty_like(q)
    if want_out:
        fpl.attn(q, k, v, out)
    res = dict(pattern=fpl.pattern.cpu().numpy(), jsd=fpl.jsd.cpu().numpy(),
               row_ptr=fpl.row_ptr.cpu().numpy(), col_idx=fpl.col_idx.cpu().numpy(),
               stats=fpl.stats(), dbg={k_: v_.numpy() for k_, v_ in fpl.debug().items()})
    if want_out:
        res["out"] = out.float().cpu().numpy()
    if dense:
        od = torch.empty_like(q)
        fpl.dense(q, k, v, od)
        res["dense"] = od.float().cpu().numpy()
    torch.cuda.synchronize()
    return res


def csr_mask(row_ptr, col_idx, nb):
    M = np.zeros((nb, nb), bool)
    for qb in range(nb):
        M[qb, col_idx[row_ptr[qb]:row_ptr[qb + 1]]] = True
    return M


def csr_rows_sorted(row_ptr, col_idx, nb):
    for qb in range(nb):
        r = col_idx[row_ptr[qb]:row_ptr[qb + 1]]
        if not (np.all(np.diff(r) > 0) and r[-1] == qb and r[0] == 0 and np.all(r <= qb)):
            return False
    return True


def classify(x, gamma, sel, delta=DELTA, lam_rel=LAM_REL):
    """Compare a GPU index set `sel` with oracle topmass(x, gamma).

    Element at oracle rank k (1-based) is selected exactly when C_{k-1} < gamma T.
    in:  C_{k-1} < gamma T - delta;   out: C_{k-1} > gamma T + delta;
    borderline: otherwise, or its score within lam_rel of the K-th score.
    Returns (missing_in, extra_out, borderline_diffs, n_borderline).
    """
    t = oracle.topmass(x, gamma)
    order, C = t["order"], t["C"]
    L = len(x)
    sel = np.asarray(sel, np.int64)
    gsel = np.zeros(L, bool)
    gsel[sel] = True
    if gamma >= 1.0:
        return int((~gsel).sum()), 0, 0, 0
    G = gamma * t["T"]
    Cprev = np.concatenate([[0.0], C[:-1]])  # C_{k-1} for rank k
    lam = x[order[t["K"] - 1]]
    xs = x[order]
    border = (np.abs(Cprev - G) <= delta) | (np.abs(xs - lam) <= lam_rel * max(lam, 1e-300))
    inn = (Cprev < G - delta) & ~border
    out = (Cprev > G + delta) & ~border
    inn[0] = inn[0] or not border[0]  # rank 1 is always selected
    g = gsel[order]
    missing_in = int((inn & ~g).sum())
    extra_out = int((out & g).sum())
    bdiff = int((border & (g != (Cprev < G))).sum())
    return missing_in, extra_out, bdiff, int(border.sum())


def oracle_inputs(q_bits, k_bits, v_bits):
    from synth import gen
    return gen.bits_to_f64(q_bits), gen.bits_to_f64(k_bits), gen.bits_to_f64(v_bits)


def rel_close(a, b, rtol, floor):
    """relative agreement on entries with |b| >= floor; absolute below."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    big = np.abs(b) >= floor
    rel = np.abs(a - b)[big] / np.abs(b)[big] if big.any() else np.zeros(1)
    small = np.abs(a - b)[~big]
    return float(rel.max(initial=0.0)), float(small.max(initial=0.0))


def stagewise_mask(pattern, dbg, h, n, gamma, min_budget, b=128, vs_mode=0, qa_mode=0,
                   max_budget=0):
    """Oracle O6-O9 (and the f1/f2 variants) applied to the GPU's own line/QA
    sets and fp32 scores.

    The budget orders are decided in fp32 like the kernel (A12 score
    a_hat[kb] + As[qb-kb] rounded to fp32; QA: A_bar in fp32). For the
    per-row QA mode the oracle's per-row topmass runs on the GPU's fp32 A_bar."""
    nb = -(-n // b)  # ragged n (A26)
    cnt = dbg["sel_count"][h]
    if pattern == oracle.VS:
        S_v = dbg["sel_v"][h, : cnt[0]]
        S_s = dbg["sel_s"][h, : cnt[1]]
        if vs_mode == 0:
            M0 = oracle.vs_block_mask(S_v, S_s, n, b)
        else:
            M0 = oracle.vs_block_mask_pooled(S_v, S_s, nb)
        ah = dbg["a_hat"][h].astype(np.float32)
        As = dbg["As"][h].astype(np.float32)
        qb = np.arange(nb)[:, None]
        kb = np.arange(nb)[None, :]
        R = (ah[kb] + As[np.clip(qb - kb, 0, nb - 1)]).astype(np.float32).astype(np.float64)
        R = np.where(kb <= qb, R, -np.inf)
    else:
        vals, rows, cols = oracle.qa_flat(np.zeros((nb, nb)))
        A = np.full((nb, nb), -np.inf)
        A[rows, cols] = dbg["A_bar"][h, : len(rows)].astype(np.float64)
        if qa_mode == 0:
            S_qa = dbg["sel_qa"][h, : cnt[2]]
            M0 = oracle.qa_block_mask(S_qa, rows, cols, nb)
        else:
            M0, _ = oracle.qa_rowwise_mask(np.where(np.isfinite(A), A, 0.0), gamma)
        R = A
    M1 = oracle.add_forced(M0)
    M2 = oracle.min_budget_extend(M1, R, min_budget, b)
    return M0, oracle.max_budget_cut(M2, R, max_budget, b)


def head_report(w, h, res, Q, K, V, qblocks, gamma=None, tau=None, min_budget=None, b=128,
                vs_mode=0, qa_mode=0, max_budget=0, near_tau=1e-4, plan=None, sel=None):
    """End-to-end parity of one head: the oracle runs from scratch on the same
    bf16 inputs (Q, K, V = this head's float64 arrays) and is compared with the
    GPU result `res` (parity.run_gpu) per SURVEY §8(c) rule 2.

    Returns a dict (printed by the tests, embedded in bench.py's parity block):
      pattern_gpu / pattern_oracle / near_tau (|D_oracle - tau| < near_tau)
      dD                 |D_gpu - D_oracle|
      sets[name]         {in_missing, out_extra, borderline, n_borderline} per
                         topmass call (a_v / a_s lines, QA flat map): the GPU set
                         must contain every "in" element and no "out" element;
                         borderline = elements within 1e-5 of the cumulative
                         threshold (or near-ties of the K-th score) whose
                         membership differs, reported separately (north_star)
      rows_equal         query-block rows whose final block lists are identical
      blocks_diff        (qb, kb) pairs selected by exactly one side
      stage_out          max / mean abs of the GPU output vs the oracle's sparse
                         attention on the GPU's CSR (sampled q-blocks)
      e2e_out            the same vs the oracle's own mask, on sampled rows whose
                         block lists match
    """
    gamma = w.gamma if gamma is None else gamma
    tau = w.tau if tau is None else tau
    min_budget = w.min_budget if min_budget is None else min_budget
    nb = -(-w.seq_len // b)
    p = oracle.plan_head(Q, K, b, tau) if plan is None else plan
    sel_o = oracle.select_head(p, Q, K, b, gamma, min_budget, vs_mode, qa_mode, max_budget) \
        if sel is None else sel
    dbg = res["dbg"]
    cnt = dbg["sel_count"][h]
    rep = dict(head=int(h), pattern_gpu=int(res["pattern"][h]), pattern_oracle=int(p["pattern"]),
               D_oracle=float(p["D"]), dD=float(abs(res["jsd"][h] - p["D"])),
               near_tau=bool(abs(p["D"] - tau) < near_tau), sets={})
    # stage (a) values: relative error on entries >= 1e-6 (SURVEY §8(c) rule 1)
    rep["plan_rel"] = max(rel_close(dbg[key][h], p[key], 1e-4, 1e-6)[0]
                          for key in ("a_v", "a_s", "a_hat", "a_bar"))
    # pooled keys (all heads) and, for QA heads, pooled queries and the pooled
    # map, normwise: max |gpu - oracle| / max |oracle|
    g = h * w.kv_heads // w.heads
    kbar = oracle.block_mean(K, b)
    rep["kbar_rel"] = float(np.abs(dbg["k_bar"][g] - kbar).max() / np.abs(kbar).max())
    if p["pattern"] == oracle.QA and res["pattern"][h] == oracle.QA:
        qbar = oracle.block_mean(Q, b)
        rep["qbar_rel"] = float(np.abs(dbg["q_bar"][h] - qbar).max() / np.abs(qbar).max())
        Ab = sel_o["Abar"] if "Abar" in sel_o else oracle.qa_pooled_map(Q, K, b)
        vals, _, _ = oracle.qa_flat(Ab)
        rep["Abar_rel"] = float(np.abs(dbg["A_bar"][h, : len(vals)] - vals).max() / np.abs(vals).max())
    if rep["pattern_gpu"] == rep["pattern_oracle"]:
        if p["pattern"] == oracle.VS:
            if vs_mode == 0:
                segs = (("a_v", p["a_v"], dbg["sel_v"][h, : cnt[0]]),
                        ("a_s", p["a_s"], dbg["sel_s"][h, : cnt[1]]))
            else:
                segs = (("a_hat", p["a_hat"], dbg["sel_v"][h, : cnt[0]]),
                        ("As", oracle.slash_block_sums(p["a_s"], b), dbg["sel_s"][h, : cnt[1]]))
        elif qa_mode == 0:
            vals, _, _ = oracle.qa_flat(sel_o["Abar"])
            segs = (("A_bar", vals, dbg["sel_qa"][h, : cnt[2]]),)
        else:
            segs = ()  # per-row QA: compared through the rows below
        for name, x, sel in segs:
            mi, eo, bd, nbd = classify(np.asarray(x, np.float64), gamma, sel)
            rep["sets"][name] = dict(in_missing=mi, out_extra=eo, borderline=bd, n_borderline=nbd)
    Mg = csr_mask(res["row_ptr"][h], res["col_idx"][h], nb)
    Mo = sel_o["mask"]
    row_eq = np.all(Mg == Mo, axis=1)
    rep["rows_equal"] = int(row_eq.sum())
    rep["config"] = f"{w.name} n={w.seq_len} gamma={gamma} tau={tau} min_budget={min_budget}" + (
        f" vs_mode={vs_mode} qa_mode={qa_mode} max_budget={max_budget}" if (vs_mode or qa_mode or max_budget) else "")
    rep["rows"] = int(nb)
    rep["blocks_diff"] = int((Mg != Mo).sum())
    if "out" in res:
        ref = oracle.sparse_attention(Q, K, V, Mg, b, qblocks)
        rows = ~np.isnan(ref[:, 0])
        d = np.abs(res["out"][h][rows] - ref[rows])
        rep["stage_out"] = dict(max_abs=float(d.max()), mean_abs=float(d.mean()))
        qb_eq = [qb for qb in qblocks if row_eq[qb]]
        if qb_eq:
            ref_e = oracle.sparse_attention(Q, K, V, Mo, b, qb_eq)
            rows_e = ~np.isnan(ref_e[:, 0])
            de = np.abs(res["out"][h][rows_e] - ref_e[rows_e])
            rep["e2e_out"] = dict(max_abs=float(de.max()), mean_abs=float(de.mean()),
                                  qblocks=len(qb_eq))
    REPORTS.append(rep)
    return rep


def check_report(rep, max_abs=2e-2, mean_abs=2e-3):
    """The north_star bar on one head_report: identical pattern (unless the
    oracle's D is within the near-tau window), |dD| <= 1e-4, no "in" element
    missing and no "out" element selected, outputs within tolerance."""
    if not rep["near_tau"]:
        assert rep["pattern_gpu"] == rep["pattern_oracle"], rep
    assert rep["dD"] <= 1e-4, rep
    assert rep["plan_rel"] <= 1e-4, rep
    assert rep["kbar_rel"] <= 1e-5, rep
    if "qbar_rel" in rep:
        assert rep["qbar_rel"] <= 1e-5, rep
        # fp32 pooled logits (|logit| up to ~10): ~1e-6 relative in the exponent
        assert rep["Abar_rel"] <= 1e-4, rep
    for name, s in rep["sets"].items():
        assert s["in_missing"] == 0 and s["out_extra"] == 0, (name, rep)
    # with no borderline membership difference (and no budget order, which the
    # GPU decides in fp32), the final block sets are identical
    if rep["pattern_gpu"] == rep["pattern_oracle"] and rep["sets"] and not budget_on(rep) \
            and all(s["borderline"] == 0 for s in rep["sets"].values()):
        assert rep["blocks_diff"] == 0, rep
    for key in ("stage_out", "e2e_out"):
        if key in rep:
            assert rep[key]["max_abs"] <= max_abs and rep[key]["mean_abs"] <= mean_abs, (key, rep)


def budget_on(rep):
    """True when a budget rule could reorder blocks (min / max budget on)."""
    return ("min_budget=0" not in rep["config"]) or ("max_budget=" in rep["config"] and "max_budget=0" not in rep["config"])
