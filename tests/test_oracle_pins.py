"""Pins for the float64 oracle (oracle/) against things other than itself.

Every oracle function is pinned by at least one of: a closed form, a library
routine (scipy / torch float64), a brute-force loop written differently, an
invariant the paper fixes, or a worked example (tests/golden/, cited). The
pins are chosen so that a dropped term, a wrong sign or index, or a
transposed operand in the oracle fails at least one of them.
"""
import itertools
import json
import math
import os

import numpy as np
import pytest
import torch
from scipy.spatial.distance import jensenshannon

import oracle
from oracle import flexprefill as F

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def rnd(seed, *shape, scale=1.0):
    return np.random.default_rng(seed).standard_normal(shape) * scale


# ------------------------------------------------------------------ O2 -------
def brute_rep_attention(Q, K, b):
    """pure-Python double loop: causal softmax of the last b rows."""
    n, d = K.shape
    out = [[0.0] * n for _ in range(b)]
    for r in range(b):
        i = n - b + r
        logits = [sum(Q[i, t] * K[j, t] for t in range(d)) / math.sqrt(d) for j in range(i + 1)]
        mx = max(logits)
        es = [math.exp(x - mx) for x in logits]
        s = sum(es)
        for j in range(i + 1):
            out[r][j] = es[j] / s
    return np.array(out)


def test_rep_attention_bruteforce_and_mask():
    Q, K = rnd(1, 24, 6), rnd(2, 24, 6)
    A = oracle.rep_attention(Q, K, 8)
    B = brute_rep_attention(Q, K, 8)
    np.testing.assert_allclose(A, B, rtol=1e-12, atol=1e-15)
    assert np.allclose(A.sum(1), 1.0)
    # entries beyond each row's position are exactly zero (P:67 causality)
    for r in range(8):
        assert np.all(A[r, 24 - 8 + r + 1:] == 0.0)


def test_rep_attention_matches_torch_softmax():
    Q, K = rnd(3, 256, 16), rnd(4, 256, 16)
    A = oracle.rep_attention(Q, K, 128)
    qt, kt = torch.tensor(Q[-128:]), torch.tensor(K)
    S = qt @ kt.T / 4.0
    mask = torch.arange(256)[None, :] > (128 + torch.arange(128))[:, None]
    ref = torch.softmax(S.masked_fill(mask, float("-inf")), dim=1).numpy()
    np.testing.assert_allclose(A, ref, rtol=1e-12, atol=1e-300)


def test_rep_attention_shift_invariance():
    # adding the same vector c to every key shifts each row's logits by q_r.c
    Q, K = rnd(5, 64, 8), rnd(6, 64, 8)
    c = rnd(7, 8)
    np.testing.assert_allclose(oracle.rep_attention(Q, K, 16), oracle.rep_attention(Q, K + c, 16),
                               rtol=1e-10, atol=1e-14)


# ------------------------------------------------------------------ O3 -------
def brute_line_scores(A, b):
    nrep, n = A.shape
    tot = 0.0
    av = [0.0] * n
    as_ = [0.0] * n
    for r in range(nrep):
        p = n - nrep + r
        for j in range(n):
            tot += A[r, j]
            av[j] += A[r, j]
            if j <= p:
                as_[p - j] += A[r, j]
    return np.array(av) / tot, np.array(as_) / tot


def test_line_scores_double_loop_tally():
    A = oracle.rep_attention(rnd(8, 64, 8), rnd(9, 64, 8), 16)
    av, as_, ah = oracle.line_scores(A, 16)
    bv, bs = brute_line_scores(A, 16)
    np.testing.assert_allclose(av, bv, rtol=1e-12, atol=1e-16)
    np.testing.assert_allclose(as_, bs, rtol=1e-12, atol=1e-16)
    assert abs(av.sum() - 1) < 1e-12 and abs(as_.sum() - 1) < 1e-12
    # a^ = blocksum(a_v) (reading A2: identical to the paper's sumpool)
    np.testing.assert_allclose(ah, av.reshape(4, 16).sum(1), rtol=1e-12)
    assert abs(ah.sum() - 1) < 1e-12


def test_line_scores_one_hot_cases():
    b, n = 4, 16
    A = np.zeros((b, n))
    A[:, 0] = 1.0  # all mass on key 0 (a sink)
    av, as_, ah = oracle.line_scores(A, b)
    assert av[0] == 1.0 and av[1:].sum() == 0
    # key 0 seen from rows at p_r = 12..15 -> offsets 12..15, each 1/4
    np.testing.assert_allclose(as_[12:16], 0.25)
    assert ah[0] == 1.0
    A = np.zeros((b, n))
    for r in range(b):
        A[r, n - b + r] = 1.0  # each row attends itself -> the main diagonal
    av, as_, ah = oracle.line_scores(A, b)
    assert as_[0] == 1.0 and as_[1:].sum() == 0
    np.testing.assert_allclose(av[n - b:], 0.25)


def test_line_scores_single_block():
    A = oracle.rep_attention(rnd(10, 8, 4), rnd(11, 8, 4), 8)
    _, _, ah = oracle.line_scores(A, 8)
    np.testing.assert_allclose(ah, [1.0])


# ------------------------------------------------------------------ O4 -------
def test_estimated_dist_equals_last_row_of_pooled_map():
    # identity: the representative set is the last query block, so
    # a_bar == N_b * A_bar[N_b - 1, :] (two different code paths in the oracle)
    Q, K = rnd(12, 128, 8), rnd(13, 128, 8)
    ab = oracle.estimated_block_dist(Q, K, 16)
    Ab = oracle.qa_pooled_map(Q, K, 16)
    np.testing.assert_allclose(ab, 8 * Ab[-1], rtol=1e-12)


def test_estimated_dist_special_cases():
    Q = rnd(14, 64, 8)
    K = np.tile(rnd(15, 1, 8), (64, 1))  # identical keys -> uniform
    np.testing.assert_allclose(oracle.estimated_block_dist(Q, K, 16), 0.25)
    np.testing.assert_allclose(oracle.estimated_block_dist(Q[:16], rnd(16, 16, 8), 16), [1.0])


def test_estimated_dist_naive():
    Q, K = rnd(17, 48, 4), rnd(18, 48, 4)
    b = 16
    qbar = [sum(Q[32 + r, t] for r in range(16)) / 16 for t in range(4)]
    kbar = [[sum(K[kb * b + r, t] for r in range(b)) / b for t in range(4)] for kb in range(3)]
    lg = [sum(qbar[t] * kbar[kb][t] for t in range(4)) / 2.0 for kb in range(3)]
    e = [math.exp(x) for x in lg]
    np.testing.assert_allclose(oracle.estimated_block_dist(Q, K, b), np.array(e) / sum(e), rtol=1e-12)


# ------------------------------------------------------------------ O5 -------
def test_js_distance_library_and_closed_forms():
    g = GOLD["js_half_vs_onehot"]
    assert abs(oracle.js_distance(g["p"], g["q"]) - g["D"]) < 1e-5
    rng = np.random.default_rng(19)
    for _ in range(20):
        p = rng.random(12) ** 3
        q = rng.random(12) ** 3
        p /= p.sum()
        q /= q.sum()
        assert abs(oracle.js_distance(p, q) - jensenshannon(p, q, base=2)) < 1e-12
        assert abs(oracle.js_distance(p, q) - oracle.js_distance(q, p)) < 1e-12
        assert oracle.js_distance(p, p) == 0.0
    assert abs(oracle.js_distance([1, 0], [0, 1]) - 1.0) < 1e-15
    # zero entries (0 log 0 = 0) on one side only
    p = np.array([0.5, 0.5, 0.0])
    q = np.array([0.2, 0.3, 0.5])
    assert abs(oracle.js_distance(p, q) - jensenshannon(p, q, base=2)) < 1e-12


def test_decide_pattern_rules():
    assert oracle.decide_pattern(0.0, 0.0) == oracle.VS  # tau = 0 -> always VS (strict <)
    assert oracle.decide_pattern(0.1, 0.1) == oracle.VS  # D == tau -> VS (A14)
    assert oracle.decide_pattern(0.0999, 0.1) == oracle.QA
    # monotone in tau
    for D in (0.01, 0.2, 0.7):
        pats = [oracle.decide_pattern(D, t) for t in np.linspace(0, 1, 41)]
        assert pats == sorted(pats)


# ------------------------------------------------------------- topmass ------
def exhaustive_min_subset(x, gamma):
    """min |S| with sum_S x >= gamma * sum x (Eq. objective), brute force."""
    L = len(x)
    T = sum(x)
    for k in range(1, L + 1):
        best = max(sum(c) for c in itertools.combinations(x, k))
        if best >= gamma * T:
            return k, best
    return L, T


@pytest.mark.parametrize("gamma", [0.3, 0.5, 0.7, 0.9, 0.95])
def test_topmass_equals_exhaustive_optimum(gamma):
    # Appendix B threshold structure: greedy top-mass is optimal
    rng = np.random.default_rng(int(gamma * 100))
    for trial in range(30):
        L = int(rng.integers(1, 13))
        x = rng.random(L) ** 4
        x /= x.sum()
        t = oracle.topmass(x, gamma)
        k, best = exhaustive_min_subset(list(x), gamma)
        assert t["K"] == k
        assert abs(t["mass"] - best) < 1e-12  # greedy prefix attains the primal optimum
        assert t["mass"] >= gamma * x.sum() - 1e-15  # coverage
        if t["K"] > 1:  # minimality: dropping the lowest selected breaks coverage
            assert t["mass"] - x[t["order"][t["K"] - 1]] < gamma * x.sum()
        # threshold structure: every selected >= every rejected
        sel = set(t["sel"].tolist())
        if 0 < len(sel) < L:
            assert min(x[list(sel)]) >= max(x[[i for i in range(L) if i not in sel]])


def test_topmass_golden_and_ties():
    for key in ("min_prefix_0.7", "min_prefix_single", "min_prefix_uniform10", "exhaustive_uniform8"):
        g = GOLD[key]
        assert oracle.topmass(g["scores"], g["gamma"])["K"] == g["K"], key
    g = GOLD["primal_dual_example"]
    t = oracle.topmass(g["scores"], g["gamma"])
    assert t["K"] == g["K"] and abs(t["mass"] - g["mass"]) < 1e-12
    assert min(np.asarray(g["scores"])[t["sel"]]) == g["threshold"]
    g = GOLD["argsort_desc"]
    assert list(oracle.topmass(g["v"], 1.0)["order"]) == g["order"]
    # equal values: ties go to the lower index (A8)
    t = oracle.topmass(np.full(8, 0.125), 0.5)
    assert list(t["sel"]) == [0, 1, 2, 3]
    x = np.array([0.1, 0.3, 0.3, 0.3])
    assert list(oracle.topmass(x, 0.5)["sel"]) == [1, 2]


def test_topmass_gamma_one_and_nesting():
    rng = np.random.default_rng(21)
    x = rng.random(50) ** 3
    x[::7] = 0.0
    assert oracle.topmass(x, 1.0)["K"] == 50  # gamma >= 1 selects everything, zeros too
    prev = set()
    for gm in (0.2, 0.5, 0.8, 0.9, 0.95, 0.99):
        s = set(oracle.topmass(x, gm)["sel"].tolist())
        assert prev <= s  # nested in gamma (same scores, same tie rule)
        prev = s
    z = np.zeros(5)
    assert oracle.topmass(z, 0.9)["K"] == 1  # gamma*T = 0 is reached by the first element


# ------------------------------------------------------------------ O6 -------
def brute_vs_blocks(S_v, S_s, n, b):
    """expand lines to element pairs, then OR into blocks."""
    nb = n // b
    M = np.zeros((nb, nb), bool)
    for i in range(n):
        for j in range(i + 1):
            if j in S_v or (i - j) in S_s:
                M[i // b, j // b] = True
    return M


def test_vs_block_mask_bruteforce():
    rng = np.random.default_rng(22)
    for trial in range(25):
        n, b = 64, 8
        S_v = set(rng.choice(n, int(rng.integers(0, 6)), replace=False).tolist())
        S_s = set(rng.choice(n, int(rng.integers(0, 6)), replace=False).tolist())
        M = oracle.vs_block_mask(sorted(S_v), sorted(S_s), n, b)
        assert np.array_equal(M, brute_vs_blocks(S_v, S_s, n, b)), (S_v, S_s)


def test_vs_block_mask_b1_is_element_level():
    # with b = 1 rasterisation is the identity, so SPEC's element examples apply
    for key in ("expand_vertical0_n4", "expand_slash0_n3", "expand_both_n3"):
        g = GOLD[key]
        M = oracle.vs_block_mask(g["verticals"], g["slashes"], g["n"], 1)
        if "pairs" in g:
            assert sorted(map(list, zip(*np.nonzero(M)))) == g["pairs"]
        else:
            assert M.sum() == g["npairs"]


# ------------------------------------------------------------------ O7 -------
def test_qa_pooled_map_naive_and_invariants():
    Q, K = rnd(23, 64, 4), rnd(24, 64, 4)
    b, nb = 16, 4
    A = oracle.qa_pooled_map(Q, K, b)
    Qb = [[sum(Q[qb * b + r, t] for r in range(b)) / b for t in range(4)] for qb in range(nb)]
    Kb = [[sum(K[kb * b + r, t] for r in range(b)) / b for t in range(4)] for kb in range(nb)]
    for qb in range(nb):
        lg = [sum(Qb[qb][t] * Kb[kb][t] for t in range(4)) / 2.0 for kb in range(qb + 1)]
        e = [math.exp(x) for x in lg]
        np.testing.assert_allclose(A[qb, : qb + 1], np.array(e) / sum(e) / nb, rtol=1e-12)
        assert np.all(A[qb, qb + 1:] == 0)
    np.testing.assert_allclose(A.sum(1), 1.0 / nb)
    Ku = np.tile(rnd(25, 1, 4), (64, 1))
    Au = oracle.qa_pooled_map(Q, Ku, b)
    for qb in range(nb):
        np.testing.assert_allclose(Au[qb, : qb + 1], 1.0 / (qb + 1) / nb)


def test_qa_flat_row_major_order():
    A = np.arange(16, dtype=float).reshape(4, 4)
    v, r, c = oracle.qa_flat(A)
    assert list(zip(r.tolist(), c.tolist())) == [(0, 0), (1, 0), (1, 1), (2, 0), (2, 1), (2, 2),
                                                 (3, 0), (3, 1), (3, 2), (3, 3)]
    assert v.tolist() == [0, 4, 5, 8, 9, 10, 12, 13, 14, 15]


# ------------------------------------------------------------------ O8, O9 ---
def test_forced_blocks():
    M = oracle.add_forced(np.zeros((5, 5), bool))
    for qb in range(5):
        assert M[qb, 0] and M[qb, qb] and M[qb].sum() == (1 if qb == 0 else 2)


def test_min_budget_extend_properties():
    rng = np.random.default_rng(26)
    nb, b = 12, 128
    for trial in range(20):
        M = np.tril(rng.random((nb, nb)) < 0.2)
        M = oracle.add_forced(M)
        R = np.where(np.tril(np.ones((nb, nb), bool)), np.round(rng.random((nb, nb)), 1), -np.inf)
        mb = int(rng.integers(1, 9)) * 128 - int(rng.integers(0, 2)) * 64
        out = oracle.min_budget_extend(M, R, mb, b)
        m = -(-mb // b)
        for qb in range(nb):
            row0, row = M[qb, : qb + 1], out[qb, : qb + 1]
            assert np.all(row >= row0)  # only adds
            assert row.sum() == max(row0.sum(), min(m, qb + 1))
            added = np.nonzero(row & ~row0)[0]
            rest = np.nonzero(~row)[0]
            for a in added:  # threshold structure with ties -> lower kb
                for z in rest:
                    assert (R[qb, a] > R[qb, z]) or (R[qb, a] == R[qb, z] and a < z)
    assert np.array_equal(oracle.min_budget_extend(M, R, 0, b), M)


def test_vs_row_scores_definition():
    a_hat = np.array([0.5, 0.3, 0.2])
    a_s = np.arange(6, dtype=float) / 15.0
    R = oracle.vs_row_scores(a_hat, a_s, 2)
    # As = [1, 5, 9] / 15 ; R[qb, kb] = a_hat[kb] + As[qb - kb]
    assert abs(R[2, 0] - (0.5 + 9 / 15)) < 1e-15
    assert abs(R[2, 1] - (0.3 + 5 / 15)) < 1e-15
    assert abs(R[1, 1] - (0.3 + 1 / 15)) < 1e-15
    assert R[0, 1] == -np.inf


# ------------------------------------------------------------- O10, O11 ------
def masked_softmax_attention(Q, K, V, E):
    """explicit -inf mask softmax with an element mask E[i, j]."""
    n, d = Q.shape
    S = Q @ K.T / math.sqrt(d)
    S = np.where(E, S, -np.inf)
    S = S - S.max(1, keepdims=True)
    P = np.exp(S)
    return (P / P.sum(1, keepdims=True)) @ V


def test_dense_matches_torch_sdpa_float64():
    Q, K, V = rnd(27, 96, 16), rnd(28, 96, 16), rnd(29, 96, 16)
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.tensor(Q)[None], torch.tensor(K)[None], torch.tensor(V)[None], is_causal=True)[0].numpy()
    np.testing.assert_allclose(oracle.dense_causal_attention(Q, K, V), ref, rtol=1e-10, atol=1e-12)


def test_sparse_attention_explicit_mask_and_full_set():
    n, b, d = 64, 8, 8
    Q, K, V = rnd(30, n, d), rnd(31, n, d), rnd(32, n, d)
    rng = np.random.default_rng(33)
    M = oracle.add_forced(np.tril(rng.random((n // b, n // b)) < 0.4))
    E = np.kron(M, np.ones((b, b), bool)) & np.tril(np.ones((n, n), bool))
    np.testing.assert_allclose(oracle.sparse_attention(Q, K, V, M, b),
                               masked_softmax_attention(Q, K, V, E), rtol=1e-10, atol=1e-12)
    full = np.tril(np.ones((n // b, n // b), bool))
    np.testing.assert_allclose(oracle.sparse_attention(Q, K, V, full, b),
                               oracle.dense_causal_attention(Q, K, V), rtol=1e-10, atol=1e-12)
    # b = 1, diagonal only -> each output row is its own V row
    np.testing.assert_allclose(oracle.sparse_attention(Q, K, V, np.eye(n, dtype=bool), 1), V, atol=1e-15)


def test_appendix_a_error_bound():
    """|A - A_S| <= (1 - a_S) sum_j |v_j| per row and dim."""
    n, b, d = 64, 8, 4
    Q, K, V = rnd(34, n, d, scale=2.0), rnd(35, n, d), rnd(36, n, d)
    rng = np.random.default_rng(37)
    M = oracle.add_forced(np.tril(rng.random((n // b, n // b)) < 0.3))
    out = oracle.sparse_attention(Q, K, V, M, b)
    dense = oracle.dense_causal_attention(Q, K, V)
    S = Q @ K.T / 2.0
    for i in range(n):
        p = np.exp(S[i, : i + 1] - S[i, : i + 1].max())
        p /= p.sum()
        sel = np.repeat(M[i // b], b)[: i + 1]
        a_S = p[sel].sum()
        bound = (1 - a_S) * np.abs(V[: i + 1]).sum(0)
        assert np.all(np.abs(dense[i] - out[i]) <= bound + 1e-12)


# ----------------------------------------------------------- pipeline --------
def test_gamma_one_reproduces_dense():
    from synth import gen
    from synth.configs import Workload
    w = Workload("t", 4, 1, 512, 1.0, 0.1, 0, 7)
    q, k, v = gen.make_layer_bits(w)
    Q, K, V = (gen.bits_to_f64(x) for x in (q, k, v))
    for h in range(4):
        r = oracle.flexprefill_head(Q[h], K[0], V[0], 128, 1.0, 0.1, 0)
        assert r["mask"].sum() == 4 * 5 // 2
        np.testing.assert_allclose(r["out"], oracle.dense_causal_attention(Q[h], K[0], V[0]),
                                   rtol=1e-10, atol=1e-12)


def test_planted_structure_is_recovered():
    """generator construction pins: pattern = planted type; sinks in S_v;
    the planted cluster blocks of the last query block are QA-selected."""
    from synth import gen
    from synth.configs import C1
    q, k, v = gen.make_layer_bits(C1)
    Q, K = gen.bits_to_f64(q), gen.bits_to_f64(k)
    meta = gen.planted(C1)[0]
    for h in range(C1.heads):
        r = oracle.flexprefill_head(Q[h], K[0], None, 128, 0.9, 0.1, 0, with_output=False)
        want = oracle.QA if gen.is_qa_type(h, C1.heads, C1.kv_heads) else oracle.VS
        assert r["pattern"] == want, (h, r["D"])
        assert abs(r["D"] - 0.1) > 0.05  # margin around tau
        if want == oracle.VS:
            assert {0, 1, 2, 3} <= set(r["S_v"].tolist())
        else:
            nb = C1.seq_len // 128
            lam = np.argmax(Q[h, -1, 102:118])
            match = [kb for kb in range(nb) if meta["clusters"][kb] == lam]
            assert all(r["mask_pre"][nb - 1, kb] for kb in match)


# ------------------------------------------------- f1 / f2 variants ----------
def brute_vs_blocks_pooled(S_vb, S_db, n, b):
    """expand vertical blocks to columns and offset groups to offsets, then the
    element pairs, then OR into blocks."""
    cols = {j for kb in S_vb for j in range(kb * b, kb * b + b)}
    offs = {o for D in S_db for o in range(D * b, min(n, D * b + b))}
    return brute_vs_blocks(cols, offs, n, b)


def test_vs_block_mask_pooled_bruteforce():
    rng = np.random.default_rng(40)
    n, b = 64, 8
    for trial in range(25):
        S_vb = sorted(set(rng.choice(8, int(rng.integers(0, 4)), replace=False).tolist()))
        S_db = sorted(set(rng.choice(8, int(rng.integers(0, 4)), replace=False).tolist()))
        M = oracle.vs_block_mask_pooled(S_vb, S_db, n // b)
        assert np.array_equal(M, brute_vs_blocks_pooled(S_vb, S_db, n, b)), (S_vb, S_db)


def test_slash_block_sums_and_pooled_equals_literal_on_aligned_offsets():
    a_s = np.arange(32, dtype=float)
    np.testing.assert_allclose(oracle.slash_block_sums(a_s, 8), [28, 92, 156, 220])
    # selecting every offset of a group at element level (R1) gives the same
    # blocks as selecting the group (R2)
    n, b = 64, 8
    for D in range(8):
        offs = list(range(D * b, D * b + b))
        assert np.array_equal(oracle.vs_block_mask([], offs, n, b),
                              oracle.vs_block_mask_pooled([], [D], n // b))


def test_qa_rowwise_mask_properties():
    Q, K = rnd(41, 128, 8), rnd(42, 128, 8)
    A = oracle.qa_pooled_map(Q, K, 16)
    for gamma in (0.5, 0.8, 0.95):
        M, per_row = oracle.qa_rowwise_mask(A, gamma)
        for qb in range(8):
            row = A[qb, : qb + 1]
            sel = np.nonzero(M[qb])[0]
            assert np.all(sel <= qb)
            assert row[sel].sum() >= gamma * row.sum() - 1e-15  # coverage per row
            k, _ = exhaustive_min_subset(list(row), gamma)  # minimality (Appendix B)
            assert len(sel) == k


def test_max_budget_cut_properties():
    rng = np.random.default_rng(43)
    nb, b = 16, 128
    for trial in range(20):
        M = oracle.add_forced(np.tril(rng.random((nb, nb)) < 0.6))
        R = np.where(np.tril(np.ones((nb, nb), bool)), np.round(rng.random((nb, nb)), 1), -np.inf)
        mb = int(rng.integers(1, 8)) * 128
        out = oracle.max_budget_cut(M, R, mb, b)
        m = -(-mb // b)
        for qb in range(nb):
            row0, row = M[qb], out[qb]
            assert np.all(row <= row0)  # only removes
            assert row[0] and row[qb]  # forced blocks survive
            cap = max(m, len({0, qb}))
            assert row.sum() == min(row0.sum(), cap)
            kept = [kb for kb in np.nonzero(row)[0] if kb not in (0, qb)]
            dropped = [kb for kb in np.nonzero(row0 & ~row)[0]]
            for a_ in kept:  # kept blocks beat dropped ones (ties -> lower kb)
                for z in dropped:
                    assert (R[qb, a_] > R[qb, z]) or (R[qb, a_] == R[qb, z] and a_ < z)
    assert np.array_equal(oracle.max_budget_cut(M, R, 0, b), M)


def test_variants_reduce_to_defaults():
    from synth import gen
    from synth.configs import C1
    q, k, v = gen.make_layer_bits(C1)
    Q, K = gen.bits_to_f64(q), gen.bits_to_f64(k)
    for h in range(C1.heads):
        p = oracle.plan_head(Q[h], K[0], 128, 0.1)
        base = oracle.select_head(p, Q[h], K[0], 128, 0.9, 0)
        big = oracle.select_head(p, Q[h], K[0], 128, 0.9, 0, max_budget=10 ** 9)
        assert np.array_equal(base["mask"], big["mask"])  # an unreachable cap changes nothing
        # gamma = 1: every variant selects every causal block
        for vm, qm in ((1, 0), (0, 1), (1, 1)):
            full = oracle.select_head(p, Q[h], K[0], 128, 1.0, 0, vs_mode=vm, qa_mode=qm)
            assert full["mask"].sum() == 16 * 17 // 2


# ------------------------------------------------- ragged n (next row f3) ----
def test_block_pooling_ragged_spec_examples():
    """sum pooling of [1,3,5,7] by 2 and avg pooling of a
    5-entry row by 2 (the ragged last cell averages its single entry)."""
    g = GOLD["block_pool_sum_1357"]
    a = np.array(g["row"], float)[None, :]
    _, _, ah = oracle.line_scores(a / a.sum(), g["block"])  # sumpool of the (1-row) map
    np.testing.assert_allclose(ah * a.sum(), g["sum"], rtol=1e-15)
    g = GOLD["block_pool_avg_ragged5"]
    X = np.array(g["row"], float)[:, None]
    np.testing.assert_allclose(F.block_mean(X, g["block"])[:, 0], g["avg"], rtol=1e-15)
    assert F.num_blocks(5, 2) == 3 and F.num_blocks(4, 2) == 2


@pytest.mark.parametrize("n,b", [(27, 8), (33, 8), (17, 16)])
def test_ragged_plan_bruteforce(n, b):
    """O2/O3/O4 on ragged n: the brute-force double loops (written without
    blocks), a^ = blocksum(a_v) over the actual keys, sum a^ = 1, and the
    naive pooled estimate with the last key block averaged over its rows."""
    d = 4
    Q, K = rnd(60 + n, n, d), rnd(61 + n, n, d)
    A = oracle.rep_attention(Q, K, b)
    np.testing.assert_allclose(A, brute_rep_attention(Q, K, b), rtol=1e-12, atol=1e-15)
    av, as_, ah = oracle.line_scores(A, b)
    bv, bs = brute_line_scores(A, b)
    np.testing.assert_allclose(av, bv, rtol=1e-12, atol=1e-16)
    np.testing.assert_allclose(as_, bs, rtol=1e-12, atol=1e-16)
    nb = -(-n // b)
    assert len(ah) == nb
    blocksum = [sum(av[j] for j in range(n) if j // b == kb) for kb in range(nb)]
    np.testing.assert_allclose(ah, blocksum, rtol=1e-12, atol=1e-17)
    assert abs(ah.sum() - 1) < 1e-12
    qbar = [sum(Q[n - b + r, t] for r in range(b)) / b for t in range(d)]
    kbar = []
    for kb in range(nb):
        rows = [j for j in range(n) if j // b == kb]
        kbar.append([sum(K[j, t] for j in rows) / len(rows) for t in range(d)])
    lg = [sum(qbar[t] * kbar[kb][t] for t in range(d)) / math.sqrt(d) for kb in range(nb)]
    e = [math.exp(x) for x in lg]
    np.testing.assert_allclose(oracle.estimated_block_dist(Q, K, b), np.array(e) / sum(e), rtol=1e-12)
    # the pooled map's last row is still a_bar / N_b (the pooled last query block
    # is the mean of its actual rows, which differs from avgpool(Q^) when ragged)
    Ab = oracle.qa_pooled_map(Q, K, b)
    np.testing.assert_allclose(Ab.sum(1), 1.0 / nb)
    Qb = [[sum(Q[i, t] for i in range(n) if i // b == qb) / len([i for i in range(n) if i // b == qb])
           for t in range(d)] for qb in range(nb)]
    for qb in range(nb):
        lg = [sum(Qb[qb][t] * kbar[kb][t] for t in range(d)) / math.sqrt(d) for kb in range(qb + 1)]
        e = [math.exp(x) for x in lg]
        np.testing.assert_allclose(Ab[qb, : qb + 1], np.array(e) / sum(e) / nb, rtol=1e-12)


def brute_vs_blocks_padded(S_v, S_s, n, b):
    """A26: lines expanded to element pairs on the b-aligned (padded) grid
    [0, N_b b)^2, then OR-ed into blocks."""
    nb = -(-n // b)
    M = np.zeros((nb, nb), bool)
    for i in range(nb * b):
        for j in range(i + 1):
            if j in S_v or (i - j) in S_s:
                M[i // b, j // b] = True
    return M


def test_vs_block_mask_ragged_bruteforce():
    rng = np.random.default_rng(62)
    for trial in range(25):
        n, b = int(rng.integers(41, 64)), 8
        S_v = set(rng.choice(n, int(rng.integers(0, 6)), replace=False).tolist())
        S_s = set(rng.choice(n, int(rng.integers(0, 6)), replace=False).tolist())
        M = oracle.vs_block_mask(sorted(S_v), sorted(S_s), n, b)
        assert np.array_equal(M, brute_vs_blocks_padded(S_v, S_s, n, b)), (n, S_v, S_s)
        if n % b == 0:
            assert np.array_equal(M, brute_vs_blocks(S_v, S_s, n, b))


def test_ragged_slash_block_sums_and_row_scores():
    a_s = np.arange(7, dtype=float)  # offsets 0..6, b = 3 -> groups [0,3), [3,6), [6,7)
    np.testing.assert_allclose(F.slash_block_sums(a_s, 3), [3.0, 12.0, 6.0])
    R = oracle.vs_row_scores(np.array([0.5, 0.3, 0.2]), a_s, 3)
    assert R[2, 0] == 0.5 + 6.0 and R[2, 2] == 0.2 + 3.0 and R[1, 2] == -np.inf


@pytest.mark.parametrize("n,b", [(27, 8), (65, 16)])
def test_ragged_sparse_attention_explicit_mask_and_bound(n, b):
    """O10 on ragged n against the explicit element mask, the full
    block set against torch SDPA (library), and the Appendix A bound."""
    d = 8
    Q, K, V = rnd(63 + n, n, d, scale=1.5), rnd(64 + n, n, d), rnd(65 + n, n, d)
    nb = -(-n // b)
    rng = np.random.default_rng(66)
    M = oracle.add_forced(np.tril(rng.random((nb, nb)) < 0.4))
    E = np.kron(M, np.ones((b, b), bool))[:n, :n] & np.tril(np.ones((n, n), bool))
    out = oracle.sparse_attention(Q, K, V, M, b)
    np.testing.assert_allclose(out, masked_softmax_attention(Q, K, V, E), rtol=1e-10, atol=1e-12)
    full = np.tril(np.ones((nb, nb), bool))
    ref = torch.nn.functional.scaled_dot_product_attention(
        torch.tensor(Q)[None], torch.tensor(K)[None], torch.tensor(V)[None], is_causal=True)[0].numpy()
    np.testing.assert_allclose(oracle.sparse_attention(Q, K, V, full, b), ref, rtol=1e-10, atol=1e-12)
    S = Q @ K.T / math.sqrt(d)
    for i in range(n):
        p = np.exp(S[i, : i + 1] - S[i, : i + 1].max())
        p /= p.sum()
        a_S = p[E[i, : i + 1]].sum()
        assert np.all(np.abs(ref[i] - out[i]) <= (1 - a_S) * np.abs(V[: i + 1]).sum(0) + 1e-12)


def test_ragged_pipeline_gamma_one_and_min_budget():
    """gamma = 1 on a ragged generated layer equals dense causal attention (SDPA
    pin above); forced blocks present; min budget fills rows to min(m, qb + 1)."""
    from synth import gen
    from synth.configs import Workload
    w = Workload("t", 2, 1, 3 * 128 + 45, 1.0, 0.1, 0, 8)
    q, k, v = gen.make_layer_bits(w)
    Q, K, V = (gen.bits_to_f64(x) for x in (q, k, v))
    for h in range(2):
        r = oracle.flexprefill_head(Q[h], K[0], V[0], 128, 1.0, 0.1, 0)
        assert r["mask"].sum() == 4 * 5 // 2
        np.testing.assert_allclose(r["out"], oracle.dense_causal_attention(Q[h], K[0], V[0]),
                                   rtol=1e-10, atol=1e-12)
        r = oracle.flexprefill_head(Q[h], K[0], V[0], 128, 0.5, 0.1, 256, with_output=False)
        for qb in range(4):
            assert r["mask"][qb, 0] and r["mask"][qb, qb]
            assert r["mask"][qb].sum() >= min(2, qb + 1)
