"""A/B timing of the host-buffer layer call (fp_layer_host) from several
library builds in one process: pinned Q/K/V -> device, plan/select/attn, O ->
host; alternating blocks of calls.

    python tools/host_ab.py lib_a.so lib_b.so [...] [--workload W]
"""
import argparse
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_20766_b200 as fp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("libs", nargs="+")
ap.add_argument("--workload", default="C3-llama8b-128k")
ap.add_argument("--blocks", type=int, default=3)
ap.add_argument("--block-len", type=int, default=4)
a = ap.parse_args()
fp.load_library()
import torch  # noqa: E402
from synth import configs, gen  # noqa: E402

w = configs.get(a.workload)
qb, kb, vb = gen.make_layer_bits(w)
qh, kh, vh = (torch.from_numpy(x).view(torch.bfloat16).pin_memory() for x in (qb, kb, vb))
oh = torch.empty_like(qh).pin_memory()
dq, dk, dv = (torch.empty(x.shape, dtype=torch.bfloat16, device="cuda") for x in (qh, kh, vh))
do = torch.empty_like(dq)
fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
P, I, Z, F = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_float
libs = []
for p in a.libs:
    L = ctypes.CDLL(os.path.abspath(p), mode=os.RTLD_LOCAL)
    L.fp_layer_host.argtypes = [P, P, P, P, P, P, P, P, I, I, I, I, I, F, F, I, P, Z, P, P, P, P, P]
    libs.append(L)
st = torch.cuda.current_stream().cuda_stream


def call(L):
    r = L.fp_layer_host(qh.data_ptr(), kh.data_ptr(), vh.data_ptr(), oh.data_ptr(), dq.data_ptr(),
                        dk.data_ptr(), dv.data_ptr(), do.data_ptr(), w.heads, w.kv_heads, w.seq_len,
                        128, 128, w.gamma, w.tau, w.min_budget, fpl.ws.data_ptr(), fpl.ws_bytes,
                        fpl.pattern.data_ptr(), fpl.jsd.data_ptr(), fpl.row_ptr.data_ptr(),
                        fpl.col_idx.data_ptr(), st)
    assert r == 0, r


outs = []
for L in libs:
    call(L)
    torch.cuda.synchronize()
    outs.append(oh.clone())
for i in range(1, len(libs)):
    print(f"lib {i}: output equal {torch.equal(outs[i], outs[0])}")
res = {p: [] for p in a.libs}
for _ in range(a.blocks):
    for p, L in zip(a.libs, libs):
        for _ in range(a.block_len):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            call(L)
            e1.record()
            torch.cuda.synchronize()
            res[p].append(e0.elapsed_time(e1))
for p in a.libs:
    print(f"{os.path.basename(p):16s} {w.name}: e2e {np.median(res[p]):.3f} ms (min {min(res[p]):.3f})")
