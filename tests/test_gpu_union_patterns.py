"""Hand-built block CSRs that stress the q-block-pair union walk of the
attention kernel (fp_attn8.cu): each CTA work item runs rows qb and qb - 1 of a
head over the UNION of their sorted block lists, with a 3-slot K ring and a
2-slot V ring whose slots are released by the entry's last PV (or early, for
the row that skips the entry). These lists make every union entry single-row
(disjoint parities) or let one row skip long runs while the other walks them,
the cases the ring release bookkeeping must survive. The reference is the
float64 oracle's block-sparse attention of the definition (P:66-83 with the
block mask M, oracle.sparse_attention), element by element at the north-star
tolerances, with and without a workspace (persistent vs one CTA per item)."""
import numpy as np
import pytest

import oracle
from tests.test_gpu_parity import MAX_ABS, MEAN_ABS

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fp():
    import paper_2502_20766_b200 as m
    m.load_library()
    return m


def _lists(kind, nb):
    """Per q-block sorted key-block lists, each ending at its diagonal block."""
    rows = []
    for r in range(nb):
        if kind == "disjoint":  # parity classes: neighbours share no block
            sel = list(range(r % 2, r, 2)) + [r]
        elif kind == "skip":  # even rows walk everything, odd rows only the diagonal
            sel = list(range(r + 1)) if r % 2 == 0 else [r]
        elif kind == "skip_other":  # odd rows walk everything, even rows only block 0 + diagonal
            sel = list(range(r + 1)) if r % 2 == 1 else sorted({0, r})
        elif kind == "sparse_far":  # a few far blocks, different per row
            sel = sorted({(7 * r + 3) % (r + 1), (r * r) % (r + 1), r})
        else:
            raise ValueError(kind)
        rows.append(np.array(sel, dtype=np.int32))
    return rows


@pytest.mark.parametrize("kind", ["disjoint", "skip", "skip_other", "sparse_far"])
@pytest.mark.parametrize("n", [2048, 2085])
def test_union_walk_matches_oracle(fp, kind, n):
    import torch
    H, G = 2, 1
    nb = -(-n // 128)
    g = torch.Generator().manual_seed(11)
    q = torch.randn(H, n, 128, generator=g).to(torch.bfloat16)
    k = torch.randn(G, n, 128, generator=g).to(torch.bfloat16)
    v = torch.randn(G, n, 128, generator=g).to(torch.bfloat16)
    qd, kd, vd = (x.cuda() for x in (q, k, v))
    rows = _lists(kind, nb)
    rp = np.zeros(nb + 1, np.int64)
    rp[1:] = np.cumsum([len(x) for x in rows])
    cap = fp.fp_col_idx_capacity(n)
    row_ptr = torch.from_numpy(np.tile(rp, (H, 1)).astype(np.int32)).cuda()
    ci = np.zeros((H, cap), np.int32)
    ci[:, :rp[-1]] = np.concatenate(rows)
    col_idx = torch.from_numpy(ci).cuda()
    ws_bytes = fp.fp_workspace_bytes(H, G, n)
    ws = torch.zeros(ws_bytes, dtype=torch.uint8, device="cuda")
    outs = {}
    for name, (w, wb) in {"ws": (ws, ws_bytes), "nows": (None, 0)}.items():
        o = torch.full_like(qd, float("nan"))
        fp.fp_sparse_attn(qd, kd, vd, o, H, G, n, row_ptr, col_idx, w, wb)
        torch.cuda.synchronize()
        outs[name] = o.float().cpu().numpy()
    assert np.array_equal(outs["ws"], outs["nows"])
    M = np.zeros((nb, nb), bool)
    for r, sel in enumerate(rows):
        M[r, sel] = True
    Q, K, V = (x.double().numpy() for x in (q, k, v))
    for h in range(H):
        ref = oracle.sparse_attention(Q[h], K[0], V[0], M, 128)
        d = np.abs(outs["ws"][h] - ref)
        assert np.isfinite(outs["ws"][h]).all()
        assert d.max() <= MAX_ABS and d.mean() <= MEAN_ABS, (kind, h, d.max(), d.mean())
