"""Per-phase clock64 breakdown of the v7 attention kernel (FP_TIMING build).

    python tools/attn7_timing.py [workload]
Softmax groups A / B (thread 0 / 128 of every 64th CTA) and the MMA issuer.
"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2502_20766_b200 as fp  # noqa: E402
from paper_2502_20766_b200 import build as B  # noqa: E402

lib_t = os.path.join(ROOT, "ab_libs", "lib_t7.so")
if not os.path.exists(lib_t) or "--rebuild" in sys.argv:
    subprocess.check_call([B.NVCC, *B.FLAGS, "-DFP_TIMING", "-DFP_ATTN_VERSION=7", "-o", lib_t] +
                          [os.path.join(B.CSRC, x) for x in B.SOURCES])
fp.load_library(lib_t)
import torch  # noqa: E402
from synth import gen, configs  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
w = configs.get(args[0] if args else "C3-llama8b-128k")
q, k, v = (torch.from_numpy(x).view(torch.bfloat16).cuda() for x in gen.make_layer_bits(w))
fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
out = torch.empty_like(q)
fpl.plan(q, k, w.tau)
fpl.select(w.gamma, w.min_budget)
fpl.attn(q, k, v, out)
torch.cuda.synchronize()
raw = ctypes.CDLL(lib_t)
buf = (ctypes.c_ulonglong * 32)()
raw.fp_debug_attn7_timing(buf, 1)
t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0.record()
fpl.attn(q, k, v, out)
t1.record()
torch.cuda.synchronize()
raw.fp_debug_attn7_timing(buf, 1)
print(f"{w.name}: attn {t0.elapsed_time(t1):.3f} ms (timing build)")
sm_names = ["wait S", "ld S+free", "softmax", "wait PV", "rescale", "st P+arrive", "-", "loop"]
for g, base in (("A", 0), ("B", 8)):
    nt = max(buf[base + 6], 1)
    tot = sum(buf[base + i] for i in (0, 1, 2, 3, 4, 5, 7))
    print(f" group {g}: {nt} sub-tiles, {tot / nt:.0f} cyc/sub-tile")
    for i in (0, 1, 2, 3, 4, 5, 7):
        print(f"   {sm_names[i]:12s} {buf[base + i] / nt:8.1f}  {100 * buf[base + i] / max(tot, 1):5.1f}%")
mma = ["wait K", "wait S free", "wait V", "wait P", "issue/other"]
ns = max(buf[16 + 5], 1)
tot = sum(buf[16 + i] for i in range(5))
print(f" MMA issuer: {ns} sub-tiles, {tot / ns:.0f} cyc/sub-tile")
for i, nm in enumerate(mma):
    print(f"   {nm:12s} {buf[16 + i] / ns:8.1f}  {100 * buf[16 + i] / max(tot, 1):5.1f}%")
