"""Interleaved A/B timing of fp_sparse_attn from several library builds loaded
into ONE process (ctypes, RTLD_LOCAL), same inputs and CSR (planned with the
first library), alternating launches so clock / power-cap drift hits all.

    python tools/attn_ab2.py lib_a.so lib_b.so [...] [--workload W] [--gamma G] [--reps 12]
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
ap.add_argument("--gamma", type=float, default=None)
ap.add_argument("--seq-len", type=int, default=None)
ap.add_argument("--reps", type=int, default=12)
ap.add_argument("--dense", action="store_true")
ap.add_argument("--block", type=int, default=128)
ap.add_argument("--blocks", type=int, default=3)
ap.add_argument("--block-len", type=int, default=12)
a = ap.parse_args()

fp.load_library(a.libs[0])
import torch  # noqa: E402
from synth import gen, configs  # noqa: E402

w = configs.get(a.workload)
if a.gamma is not None:
    w = w.with_(gamma=a.gamma)
if a.seq_len is not None:
    w = w.with_(seq_len=a.seq_len)
q, k, v = (torch.from_numpy(x).view(torch.bfloat16).cuda() for x in gen.make_layer_bits(w))
fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len, block_size=a.block)
out = torch.empty_like(q)
fpl.plan(q, k, w.tau)
fpl.select(w.gamma, w.min_budget)
libs = []
for p in a.libs:
    L = ctypes.CDLL(os.path.abspath(p), mode=os.RTLD_LOCAL)
    P, I, Z = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
    L.fp_sparse_attn.argtypes = [P, P, P, P, I, I, I, I, I, P, P, P, Z, P]
    L.fp_dense_causal_attn.argtypes = [P, P, P, P, I, I, I, I, I, P, Z, P]
    libs.append(L)
st = torch.cuda.current_stream().cuda_stream


def call(L):
    if a.dense:
        r = L.fp_dense_causal_attn(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), w.heads,
                                   w.kv_heads, w.seq_len, 128, 128, fpl.ws.data_ptr(), fpl.ws_bytes, st)
    else:
        r = L.fp_sparse_attn(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), w.heads,
                             w.kv_heads, w.seq_len, 128, a.block, fpl.row_ptr.data_ptr(),
                             fpl.col_idx.data_ptr(), fpl.ws.data_ptr(), fpl.ws_bytes, st)
    assert r == 0, r


ref = []
for L in libs:
    call(L)
    torch.cuda.synchronize()
    ref.append(out.clone())
for i in range(1, len(libs)):
    d = (ref[i].float() - ref[0].float()).abs().max().item()
    print(f"max |out[{i}] - out[0]| = {d:.3e}")
times = [[] for _ in libs]
for r in range(a.reps):
    for i, L in enumerate(libs):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call(L)
        e1.record()
        torch.cuda.synchronize()
        times[i].append(e0.elapsed_time(e1))
for p, t in zip(a.libs, times):
    t = np.array(t)
    print(f"{os.path.basename(p):18s} {w.name} g={w.gamma}: median {np.median(t):.3f} ms  min {t.min():.3f}  max {t.max():.3f}")

# alternating BLOCKS of back-to-back launches (the power-cap clock settles
# within a block, as in bench.py's timed steps), SM clock / board power
# sampled during each block (nvidia-smi, 100 ms): a power-capped kernel shows
# the clock down and the power at the cap, a latency-bound one neither.
from bench import ClockSampler  # noqa: E402
bt = [[] for _ in libs]
bclk = [[] for _ in libs]
bpw = [[] for _ in libs]
for b in range(a.blocks):
    for i, L in enumerate(libs):
        with ClockSampler(torch.cuda.current_device()) as cs:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(a.block_len):
                call(L)
            e1.record()
            torch.cuda.synchronize()
        bt[i].append(e0.elapsed_time(e1) / a.block_len)
        for ln in cs.lines:
            f = ln.split(",")
            try:
                bclk[i].append(float(f[0]))
                bpw[i].append(float(f[2]))
            except (ValueError, IndexError):
                pass
for p, t, c, pw in zip(a.libs, bt, bclk, bpw):
    print(f"{os.path.basename(p):18s} blocks: median {np.median(t):.3f} ms/launch  min {min(t):.3f}  "
          f"sm {np.median(c) if c else None} MHz  power {np.median(pw) if pw else None} W")
