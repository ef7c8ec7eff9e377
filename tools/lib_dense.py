"""Context measurement: this library's dense causal kernel (fp_dense_causal_attn) beside the
vendor dense attention kernels available in the image (torch SDPA with the cuDNN and the
flash backends), same bf16 inputs, same GPU, alternating blocks of launches so the power-capped
clock hits every arm alike. Not on the product path; it tells whether the dense/sparse kernels'
~1.2 PFLOP/s is a kernel limit or the chip's limit under the power cap.

    python tools/lib_dense.py [--seq 32768 131072] [--heads 32] [--kv-heads 8] [--block-len 6]
Prints one JSON line per (seq, arm).
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import torch.nn.functional as F  # noqa: E402
from torch.nn.attention import SDPBackend, sdpa_kernel  # noqa: E402

import paper_2502_20766_b200 as fp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, nargs="+", default=[32768, 131072])
ap.add_argument("--heads", type=int, default=32)
ap.add_argument("--kv-heads", type=int, default=8)
ap.add_argument("--blocks", type=int, default=3)
ap.add_argument("--block-len", type=int, default=6)
ap.add_argument("--arms", nargs="+", default=None)
a = ap.parse_args()

fp.load_library()
H, G, D = a.heads, a.kv_heads, 128


class Clocks:
    def __init__(self):
        self.s, self.stop = [], False

    def run(self):
        while not self.stop:
            try:
                r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw",
                                    "--format=csv,noheader,nounits", "-i", "0"],
                                   capture_output=True, text=True, timeout=5).stdout
                mhz, w = r.strip().split("\n")[0].split(",")
                self.s.append((float(mhz), float(w)))
            except Exception:
                pass
            time.sleep(0.2)


for n in a.seq:
    g = torch.Generator(device="cuda").manual_seed(n)
    q = torch.randn(H, n, D, device="cuda", dtype=torch.bfloat16, generator=g)
    k = torch.randn(G, n, D, device="cuda", dtype=torch.bfloat16, generator=g)
    v = torch.randn(G, n, D, device="cuda", dtype=torch.bfloat16, generator=g)
    o = torch.empty_like(q)
    fpl = fp.FlexPrefill(H, G, n)
    useful = 4.0 * D * H * (n * (n + 1) / 2)  # causal QK^T + PV, multiply-add = 2 FLOP
    kr = k.repeat_interleave(H // G, 0).unsqueeze(0)
    vr = v.repeat_interleave(H // G, 0).unsqueeze(0)
    q4 = q.unsqueeze(0)

    def ours():
        fpl.dense(q, k, v, o)

    def sdpa(backend):
        def f():
            with sdpa_kernel([backend]):
                F.scaled_dot_product_attention(q4, kr, vr, is_causal=True)
        return f

    arms = {"fp_dense_causal_attn": ours, "sdpa_cudnn": sdpa(SDPBackend.CUDNN_ATTENTION),
            "sdpa_flash": sdpa(SDPBackend.FLASH_ATTENTION)}
    if a.arms:
        arms = {k_: f for k_, f in arms.items() if k_ in a.arms}
    ok = {}
    ref = None
    for name, f in arms.items():
        try:
            f()
            torch.cuda.synchronize()
            ok[name] = f
        except Exception as e:  # backend not available for this shape / arch
            print(json.dumps({"seq": n, "arm": name, "unavailable": str(e).split("\n")[0][:200]}),
                  flush=True)
    # agreement check on a slice (the cuDNN arm is the comparison, not an oracle)
    with sdpa_kernel([SDPBackend.CUDNN_ATTENTION]):
        try:
            if a.arms:
                raise RuntimeError("skipped")
            ref = F.scaled_dot_product_attention(q4, kr, vr, is_causal=True)[0]
            ours()
            torch.cuda.synchronize()
            diff = (o.float() - ref.float()).abs()
            print(json.dumps({"seq": n, "ours_vs_cudnn_maxabs": diff.max().item(),
                              "mean": diff.mean().item()}), flush=True)
        except Exception:
            pass
    del ref
    times = {k_: [] for k_ in ok}
    clk = {k_: Clocks() for k_ in ok}
    for _ in range(a.blocks):
        for name, f in ok.items():
            th = threading.Thread(target=clk[name].run, daemon=True)
            clk[name].stop = False
            th.start()
            f()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(a.block_len):
                f()
            e1.record()
            torch.cuda.synchronize()
            clk[name].stop = True
            th.join()
            times[name].append(e0.elapsed_time(e1) / a.block_len)
    for name in ok:
        ms = sorted(times[name])[len(times[name]) // 2]
        s = clk[name].s
        mhz = sorted(x[0] for x in s)[len(s) // 2] if s else None
        wat = sorted(x[1] for x in s)[len(s) // 2] if s else None
        print(json.dumps({"seq": n, "heads": H, "kv_heads": G, "arm": name, "ms": ms,
                          "all_ms": times[name], "tflops_useful": useful / ms / 1e9,
                          "sm_mhz_median": mhz, "power_w_median": wat}), flush=True)
    del q, k, v, o, kr, vr, q4, fpl
    torch.cuda.empty_cache()
