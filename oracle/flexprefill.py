"""Plain float64 implementation of FlexPrefill (O1..O11).

TEST INFRASTRUCTURE -- see oracle/__init__.py. Slow and obvious on purpose:
each function is one step of Alg. 1-4 of the paper written in the
paper's order and notation, using numpy float64 on the exact values of the
bf16 inputs. No blocking, fusion or reordering beyond what the definitions
state. Readings of silent / ambiguous passages are tagged A1..A26.
"""
import math
import numpy as np

QA = 1  # query_specific (Alg. 2)
VS = 0  # vertical_slash (Alg. 2)


# ---------------------------------------------------------------- O1, O2 -----
def representative_queries(Qh, b):
    """O1: Q^ = Q[-block_size:]  ("the last block_size query vectors")."""
    return Qh[Qh.shape[0] - b:]


def rep_attention(Qh, Kg, b):
    """O2: A^ = softmax(Q^ K^T / sqrt(d)) over the causally visible keys.

    P:348 (Alg. 3 line 1) and P:192 (the softmax inside a^). Row r is the
    query at global position p_r = n - b + r; keys j > p_r are masked (P:67,
    S_i subset of {j <= i}; reading A4). Scale 1/sqrt(d) (A16).
    Returns A^ with shape (b, n); row r sums to 1.
    """
    n, d = Kg.shape
    Qhat = representative_queries(Qh, b)
    S = (Qhat @ Kg.T) / math.sqrt(d)
    p = n - b + np.arange(b)
    S[np.arange(n)[None, :] > p[:, None]] = -np.inf
    S = S - S.max(axis=1, keepdims=True)
    E = np.exp(S)
    return E / E.sum(axis=1, keepdims=True)


# -------------------------------------------------------------------- O3 -----
def line_scores(Ahat, b):
    """O3: vertical and slash line scores, and the true block distribution a^.

    a_v = sum_vertical(A^) / sum A^
    a_s = sum_slash(A^)    / sum A^              (A9: offset o = p_r - j)
    a^  = sumpool(softmax(Q^ K^T/sqrt d))        (A2: the mean over the
          b rows of each row's key-block mass, which is blocksum(a_v))
    Returns (a_v[n], a_s[n], a_hat[n/b]).
    """
    nrep, n = Ahat.shape
    total = Ahat.sum()
    a_v = Ahat.sum(axis=0) / total
    a_s = np.zeros(n)
    for r in range(nrep):
        p_r = n - nrep + r
        # offsets o = 0..p_r pick A^[r, p_r - o]
        a_s[: p_r + 1] += Ahat[r, p_r::-1]
    a_s /= total
    # sumpool over key blocks of each row's softmax, averaged over the b rows (A2);
    # a ragged last block (n % b != 0) is pooled over its actual keys (A26)
    nb = num_blocks(n, b)
    a_hat = np.array([Ahat[:, kb * b:(kb + 1) * b].sum(axis=1).mean() for kb in range(nb)])
    return a_v, a_s, a_hat


# -------------------------------------------------------------------- O4 -----
def num_blocks(n, b):
    """N_b = ceil(n / b): a ragged last block holds the n mod b trailing positions (A26)."""
    return -(-n // b)


def block_mean(X, b):
    """avgpool with kernel = stride = block_size along the sequence (A3);
    a ragged last block averages over its actual rows (A26)."""
    n, d = X.shape
    return np.array([X[kb * b:(kb + 1) * b].mean(axis=0) for kb in range(num_blocks(n, b))])


def estimated_block_dist(Qh, Kg, b):
    """O4: a_bar = softmax(avgpool(Q^) avgpool(K)^T / sqrt(d)).

    avgpool(Q^) is a single pooled query (Q^ is one block). No mask across the
    N_b pooled keys (A4: every key block is visible from the last query block).
    """
    d = Kg.shape[1]
    qbar = representative_queries(Qh, b).mean(axis=0)
    logits = block_mean(Kg, b) @ qbar / math.sqrt(d)
    logits = logits - logits.max()
    e = np.exp(logits)
    return e / e.sum()


# -------------------------------------------------------------------- O5 -----
def js_distance(p, q):
    """D_JS = sqrt(JSD(p||q)) = sqrt(1/2 (KL(p||m) + KL(q||m))), m = (p+q)/2.

    Eq. js_distance. Base-2 logarithms (A1) so D in [0, 1];
    0 log 0 = 0; JSD clamped at 0 before the square root (A14).
    """
    p = np.asarray(p, np.float64)
    q = np.asarray(q, np.float64)
    m = 0.5 * (p + q)

    def kl(a, c):
        nz = a > 0
        return float(np.sum(a[nz] * np.log2(a[nz] / c[nz])))

    jsd = 0.5 * (kl(p, m) + kl(q, m))
    return math.sqrt(max(0.0, jsd))


def decide_pattern(D, tau):
    """Alg. 2: query_specific iff d_JS < tau, else vertical_slash (A14)."""
    return QA if D < tau else VS


# ------------------------------------------------------------- topmass -------
def topmass(x, gamma):
    """Cumulative-attention selection (Alg. 3, Alg. 4).

    I = argsort(x) descending, ties -> lower index (A8);
    K = min{k : sum_{i in I[1:k]} x[i] >= gamma * T}, T = sum x (A6, A7);
    gamma >= 1 selects everything (A7). Returns dict with the selected
    indices in ascending order, K, the achieved mass C_K, and the sort order
    and prefix sums (for the borderline classifier).
    """
    x = np.asarray(x, np.float64)
    L = x.shape[0]
    order = np.lexsort((np.arange(L), -x))
    C = np.cumsum(x[order])
    T = C[-1] if L else 0.0
    if gamma >= 1.0:
        K = L
    else:
        K = int(np.searchsorted(C, gamma * T, side="left")) + 1
        K = min(K, L)
    sel = np.sort(order[:K])
    return dict(sel=sel, K=K, mass=float(C[K - 1]) if K else 0.0, order=order, C=C, T=float(T))


# -------------------------------------------------------------------- O6 -----
def vs_block_mask(S_v, S_s, n, b):
    """O6: extend the selected lines to the whole attention matrix, at
    block granularity (A10, reading R1).

    vertical j   -> key-block column floor(j/b), for every query block >= it;
    slash o      -> block diagonals floor(o/b), and floor(o/b)+1 if o mod b != 0
                    (a slash at offset o crosses those two block diagonals);
    block (qb, kb <= qb) is selected iff kb in Vb or qb - kb in Db.
    For ragged n the rule is applied on the b-aligned block grid (A26).
    """
    nb = num_blocks(n, b)
    Vb = np.zeros(nb, bool)
    Vb[np.asarray(S_v, np.int64) // b] = True
    Db = np.zeros(nb + 1, bool)
    S_s = np.asarray(S_s, np.int64)
    Db[S_s // b] = True
    Db[(S_s // b + 1)[S_s % b != 0]] = True
    qb = np.arange(nb)[:, None]
    kb = np.arange(nb)[None, :]
    causal = kb <= qb
    delta = np.clip(qb - kb, 0, nb)
    return causal & (Vb[kb] | Db[delta])


# -------------------------------------------------------------------- O7 -----
def qa_pooled_map(Qh, Kg, b):
    """O7 (first half): A_bar = softmax(pool(Q) pool(K)^T / sqrt(d)), flattened
    and normalised (Alg. 4).

    avgpool Q and K per block (A3); row-wise softmax over the causally visible
    key blocks kb <= qb (A4, A5); then A_bar / sum(A_bar).
    Returns the (N_b, N_b) map with zeros above the diagonal.
    """
    n, d = Kg.shape
    nb = num_blocks(n, b)
    L = block_mean(Qh, b) @ block_mean(Kg, b).T / math.sqrt(d)
    A = np.zeros((nb, nb))
    for qb in range(nb):
        row = L[qb, : qb + 1]
        e = np.exp(row - row.max())
        A[qb, : qb + 1] = e / e.sum()
    return A / A.sum()


def qa_flat(Abar):
    """flatten over the causal entries, row-major: flat index qb*N_b + kb (A8).

    Returns (values, rows, cols) in that order.
    """
    nb = Abar.shape[0]
    rows, cols = np.tril_indices(nb)
    return Abar[rows, cols], rows, cols


def qa_block_mask(sel, rows, cols, nb):
    """S = I_a[1:K] as a block mask."""
    M = np.zeros((nb, nb), bool)
    M[rows[sel], cols[sel]] = True
    return M


# ------------------------------------------------------------------ O8, O9 ---
def add_forced(M):
    """O8: retain the first and last key blocks of each query block (A11)."""
    M = M.copy()
    nb = M.shape[0]
    M[:, 0] = True
    M[np.arange(nb), np.arange(nb)] = True
    return M


def vs_row_scores(a_hat, a_s, b):
    """Row score used by the VS minimum-budget extension (A12):
    score(qb, kb) = a^[kb] + As[qb - kb], As[D] = sum of a_s over [D b, (D+1) b)."""
    nb = a_hat.shape[0]
    As = slash_block_sums(a_s, b)
    qb = np.arange(nb)[:, None]
    kb = np.arange(nb)[None, :]
    R = a_hat[kb] + As[np.clip(qb - kb, 0, nb - 1)]
    return np.where(kb <= qb, R, -np.inf)


def min_budget_extend(M, R, min_budget, b):
    """O9: each attention head computes at least `min_budget` tokens.

    Reading A12: per query-block row, at least m = ceil(min_budget / b) key
    blocks (clamped to qb + 1); missing blocks are the best unselected
    kb <= qb by row score R (descending), ties -> lower kb.
    """
    if min_budget <= 0:
        return M.copy()
    M = M.copy()
    nb = M.shape[0]
    m = -(-min_budget // b)
    for qb in range(nb):
        need = min(m, qb + 1) - int(M[qb, : qb + 1].sum())
        if need <= 0:
            continue
        cand = [kb for kb in range(qb + 1) if not M[qb, kb]]
        cand.sort(key=lambda kb: (-R[qb, kb], kb))
        for kb in cand[:need]:
            M[qb, kb] = True
    return M


# --------------------------------------------- next rows f1 / f2 (variants) ---
def slash_block_sums(a_s, b):
    """As[D] = sum of a_s over offsets [D b, (D+1) b) (the A12 row-score term);
    the last group holds the offsets < n only (A26)."""
    nb = num_blocks(a_s.shape[0], b)
    return np.array([a_s[D * b:(D + 1) * b].sum() for D in range(nb)])


def vs_block_mask_pooled(S_vb, S_db, nb):
    """f1, reading R2 (block-pooled lines): vertical *blocks* S_vb selected by
    topmass(a_hat), slash *offset groups* S_db selected by topmass(As). The
    offsets of group D = [D b, (D+1) b) lie on block diagonals D and D+1 (an
    element pair (i, i-o) with o in the group has floor(i/b) - floor((i-o)/b)
    in {D, D+1}), so a selected group marks both; block (qb, kb <= qb) is
    selected iff kb in S_vb or qb - kb in {D, D+1 : D in S_db}."""
    Vb = np.zeros(nb, bool)
    Vb[np.asarray(S_vb, np.int64)] = True
    Db = np.zeros(nb + 1, bool)
    S_db = np.asarray(S_db, np.int64)
    Db[S_db] = True
    Db[S_db + 1] = True
    qb = np.arange(nb)[:, None]
    kb = np.arange(nb)[None, :]
    return (kb <= qb) & (Vb[kb] | Db[np.clip(qb - kb, 0, nb)])


def qa_rowwise_mask(Abar, gamma):
    """f2 "wo/ flatten": per query block, the smallest set of key
    blocks whose pooled-estimate mass reaches gamma of that row's mass (the
    topmass rule of Alg. 4 applied to each row of A_bar instead of the
    flattened map). Returns (mask, list of per-row topmass results)."""
    nb = Abar.shape[0]
    M = np.zeros((nb, nb), bool)
    per_row = []
    for qb in range(nb):
        t = topmass(Abar[qb, : qb + 1], gamma)
        M[qb, t["sel"]] = True
        per_row.append(t)
    return M, per_row


def max_budget_cut(M, R, max_budget, b):
    """f2 maximum budget, read like A12: per query-block row at
    most m = ceil(max_budget / b) key blocks; rows above the cap keep their
    forced blocks {0, qb} (never removed) and then the best remaining
    selected blocks by row score R (descending, ties -> lower kb)."""
    if max_budget <= 0:
        return M.copy()
    M = M.copy()
    nb = M.shape[0]
    m = -(-max_budget // b)
    for qb in range(nb):
        sel = [kb for kb in range(qb + 1) if M[qb, kb]]
        forced = {0, qb}
        cap = max(m, len(forced))
        if len(sel) <= cap:
            continue
        keep = set(forced)
        rest = sorted((kb for kb in sel if kb not in forced), key=lambda kb: (-R[qb, kb], kb))
        keep.update(rest[: cap - len(forced)])
        M[qb, :] = False
        M[qb, sorted(keep)] = True
    return M


# ------------------------------------------------------------- O10, O11 ------
def sparse_attention(Qh, Kg, Vg, M, b, qblocks=None):
    """O10: y = A(Q, K, V, S) = softmax((Q K^T + M_S)/sqrt d) V.

    S is the block mask M intersected with the causal set j <= i.
    Returns the (n, d) output (rows of q-blocks not in `qblocks` left NaN).
    """
    n, d = Qh.shape
    nb = num_blocks(n, b)
    out = np.full((n, d), np.nan)
    for qb in range(nb) if qblocks is None else qblocks:
        kbs = np.nonzero(M[qb, : qb + 1])[0]
        keys = (kbs[:, None] * b + np.arange(b)[None, :]).reshape(-1)
        keys = keys[keys < n]  # ragged last block (A26)
        qi = np.arange(qb * b, min((qb + 1) * b, n))
        S = Qh[qi] @ Kg[keys].T / math.sqrt(d)
        S[keys[None, :] > qi[:, None]] = -np.inf
        S = S - S.max(axis=1, keepdims=True)
        P = np.exp(S)
        P /= P.sum(axis=1, keepdims=True)
        out[qi] = P @ Vg[keys]
    return out


def dense_causal_attention(Qh, Kg, Vg):
    """O11: full causal attention A(Q, K, V)."""
    n, d = Qh.shape
    S = Qh @ Kg.T / math.sqrt(d)
    S[np.triu_indices(n, 1)] = -np.inf
    S = S - S.max(axis=1, keepdims=True)
    P = np.exp(S)
    P /= P.sum(axis=1, keepdims=True)
    return P @ Vg


# ---------------------------------------------------------- orchestration ----
def plan_head(Qh, Kg, b, tau):
    """Alg. 2 (Sparse Pattern Search) plus the VS line scores of
    Alg. 3 computed from the same A^ (reading A20)."""
    Ahat = rep_attention(Qh, Kg, b)
    a_v, a_s, a_hat = line_scores(Ahat, b)
    a_bar = estimated_block_dist(Qh, Kg, b)
    D = js_distance(a_bar, a_hat)
    return dict(pattern=decide_pattern(D, tau), D=D, a_v=a_v, a_s=a_s, a_hat=a_hat, a_bar=a_bar)


def select_head(plan, Qh, Kg, b, gamma, min_budget, vs_mode=0, qa_mode=0, max_budget=0):
    """Alg. 3 or Alg. 4 by pattern, then forced blocks (O8), minimum budget (O9)
    and maximum budget (f2). vs_mode 1 = block-pooled lines (f1, R2);
    qa_mode 1 = per-query-block selection (f2, "wo/ flatten")."""
    n = Kg.shape[0]
    nb = num_blocks(n, b)
    out = dict()
    if plan["pattern"] == VS:
        if vs_mode == 0:
            tv = topmass(plan["a_v"], gamma)
            ts = topmass(plan["a_s"], gamma)
            M0 = vs_block_mask(tv["sel"], ts["sel"], n, b)
        else:
            tv = topmass(plan["a_hat"], gamma)
            ts = topmass(slash_block_sums(plan["a_s"], b), gamma)
            M0 = vs_block_mask_pooled(tv["sel"], ts["sel"], nb)
        out.update(tv=tv, ts=ts, S_v=tv["sel"], S_s=ts["sel"])
        R = vs_row_scores(plan["a_hat"], plan["a_s"], b)
    else:
        Abar = qa_pooled_map(Qh, Kg, b)
        if qa_mode == 0:
            vals, rows, cols = qa_flat(Abar)
            tq = topmass(vals, gamma)
            out.update(tq=tq, S_qa=tq["sel"])
            M0 = qa_block_mask(tq["sel"], rows, cols, nb)
        else:
            M0, per_row = qa_rowwise_mask(Abar, gamma)
            out.update(tq_rows=per_row)
        out.update(Abar=Abar)
        R = np.where(np.tril(np.ones((nb, nb), bool)), Abar, -np.inf)
    M1 = add_forced(M0)
    M2 = min_budget_extend(M1, R, min_budget, b)
    M = max_budget_cut(M2, R, max_budget, b)
    out.update(mask_pre=M0, mask_forced=M1, mask_min=M2, mask=M, row_score=R)
    return out


def flexprefill_head(Qh, Kg, Vg, b=128, gamma=0.9, tau=0.1, min_budget=0, qblocks=None,
                     with_output=True, vs_mode=0, qa_mode=0, max_budget=0):
    """Alg. 1 (Sparse Attention) for one Q head."""
    plan = plan_head(Qh, Kg, b, tau)
    sel = select_head(plan, Qh, Kg, b, gamma, min_budget, vs_mode, qa_mode, max_budget)
    res = dict(plan)
    res.update(sel)
    if with_output:
        res["out"] = sparse_attention(Qh, Kg, Vg, sel["mask"], b, qblocks)
    return res
