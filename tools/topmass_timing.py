"""Phase timeline of topmass_kernel (build with -DFP_TM_TIMING): globaltimer
stamps of thread 0 per CTA, averaged per head pattern.

    python tools/topmass_timing.py lib.so [--workload W]
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
ap.add_argument("lib")
ap.add_argument("--workload", default="C3-llama8b-128k")
a = ap.parse_args()
fp.load_library(a.lib)
import torch  # noqa: E402
from synth import configs, gen  # noqa: E402

w = configs.get(a.workload)
q, k, v = (torch.from_numpy(x).view(torch.bfloat16).cuda() for x in gen.make_layer_bits(w))
fpl = fp.FlexPrefill(w.heads, w.kv_heads, w.seq_len)
fpl.plan(q, k, w.tau)
for _ in range(3):
    fpl.select(w.gamma, w.min_budget)
torch.cuda.synchronize()
L = ctypes.CDLL(os.path.abspath(a.lib), mode=os.RTLD_LOCAL)
buf = np.zeros((512, 16), dtype=np.uint64)
assert L.fp_debug_topmass_timing(buf.ctypes.data_as(ctypes.c_void_p)) == 0
pat = fpl.pattern.cpu().numpy()
t0 = min(int(x) for x in buf[:, 0] if x)
names = ["zero", "hist", "merge", "scan"]
for kind, sel in (("QA", 1), ("VS", 0)):
    rows = [buf[h * 8 + r] for h in range(w.heads) if pat[h] == sel for r in range(8) if buf[h * 8 + r, 0]]
    if not rows:
        continue
    R = np.array(rows, dtype=np.float64)
    print(f"{kind}: {len(rows)} CTAs; start {np.mean(R[:, 0] - t0) / 1e3:.1f} us after the first, "
          f"end {np.mean(R[:, 15] - t0) / 1e3:.1f} us (max {np.max(R[:, 15] - t0) / 1e3:.1f})")
    prev = R[:, 0]
    for p in range(3):
        for j, nm in enumerate(names):
            col = R[:, 1 + 4 * p + j]
            print(f"  pass {p} {nm:5s} {np.mean(col - prev) / 1e3:7.2f} us")
            prev = col
    for nm, c in (("offsets", 13), ("compact", 14), ("exit", 15)):
        print(f"  {nm:12s} {np.mean(R[:, c] - prev) / 1e3:7.2f} us")
        prev = R[:, c]
