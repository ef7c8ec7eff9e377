"""Where do two library builds disagree? Runs fp_sparse_attn (or dense) from two .so files
on the same inputs/CSR and prints the worst (head, q-block) cells and a per-q-block profile.

    python tools/ab_diff.py lib_ref.so lib_new.so [--workload W] [--dense]
"""
import argparse
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_20766_b200 as fp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs=2)
ap.add_argument("--workload", default="C2-llama8b-32k")
ap.add_argument("--dense", action="store_true")
a = ap.parse_args()
fp.load_library(os.path.abspath(a.libs[0]))
import torch  # noqa: E402
from synth import gen, configs  # noqa: E402

w = configs.get(a.workload)
q, k, v = (torch.from_numpy(x).view(torch.bfloat16).cuda() for x in gen.make_layer_bits(w))
fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
fpl.plan(q, k, w.tau)
fpl.select(w.gamma, w.min_budget)
outs = []
P, I, Z = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
st = torch.cuda.current_stream().cuda_stream
for p in a.libs:
    L = ctypes.CDLL(os.path.abspath(p), mode=os.RTLD_LOCAL)
    L.fp_sparse_attn.argtypes = [P, P, P, P, I, I, I, I, I, P, P, P, Z, P]
    L.fp_dense_causal_attn.argtypes = [P, P, P, P, I, I, I, I, I, P, Z, P]
    out = torch.zeros_like(q)
    if a.dense:
        r = L.fp_dense_causal_attn(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), w.heads,
                                   w.kv_heads, w.seq_len, 128, 128, None, 0, st)
    else:
        r = L.fp_sparse_attn(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), w.heads,
                             w.kv_heads, w.seq_len, 128, 128, fpl.row_ptr.data_ptr(),
                             fpl.col_idx.data_ptr(), fpl.ws.data_ptr(), fpl.ws_bytes, st)
    assert r == 0, r
    torch.cuda.synchronize()
    outs.append(out.float())
nb = (w.seq_len + 127) // 128
d = (outs[0] - outs[1]).abs()
d = torch.nn.functional.pad(d, (0, 0, 0, nb * 128 - w.seq_len)).view(w.heads, nb, 128, 128)
cell = d.amax(dim=(2, 3))  # [H, nb]
print("max", cell.max().item(), "bad cells (>0.05):", int((cell > 0.05).sum()), "of", cell.numel())
bad = (cell > 0.05).nonzero().tolist()
print("first bad (h, qb):", bad[:20])
print("bad per parity of qb (row A = odd qb when nb even):",
      {p: int((cell[:, p::2] > 0.05).sum()) for p in (0, 1)})
rowd = d.amax(dim=3)  # [H, nb, 128]
if bad:
    h, qb = bad[0]
    print("rows of first bad cell with err > 0.05:", (rowd[h, qb] > 0.05).nonzero().flatten().tolist()[:40])
    print("row-in-block error profile over all bad cells (count > 0.05 per row idx, 16-groups):",
          [(int((rowd[:, :, g * 16:(g + 1) * 16] > 0.05).sum())) for g in range(8)])
