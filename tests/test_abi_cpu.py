"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/flexprefill.h declares, sizes workspaces, and validates arguments
(every validation error is returned before any device work is attempted)."""
import ctypes
import os
import re

import pytest

import paper_2502_20766_b200 as fp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "flexprefill.h")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(fp.LIB_PATH):
        from paper_2502_20766_b200 import build
        build.build()
    return fp.load_library()


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fp_[a-z_]+)\s*\(", src)))


def test_exports_every_declared_symbol(lib):
    syms = declared_symbols()
    assert {"fp_plan", "fp_select", "fp_sparse_attn", "fp_dense_causal_attn"} <= set(syms)
    raw = ctypes.CDLL(fp.LIB_PATH)
    for s in syms:
        assert hasattr(raw, s), s


def test_workspace_and_capacity(lib):
    assert fp.fp_col_idx_capacity(131072) == 1024 * 1025 // 2
    b1 = fp.fp_workspace_bytes(32, 8, 32768)
    b2 = fp.fp_workspace_bytes(32, 8, 131072)
    assert 0 < b1 < b2 < (1 << 31)
    for bad in [(32, 7, 32768), (32, 8, 100), (32, 8, 64), (0, 1, 2048)]:
        assert fp.fp_workspace_bytes(*bad) == 0
    assert fp.fp_workspace_bytes(4, 1, 2048, head_dim=64) == 0
    # block_size 64 (next row f3): supported; other sizes are not
    b64 = fp.fp_workspace_bytes(4, 1, 2048, block_size=64)
    assert b64 > fp.fp_workspace_bytes(4, 1, 2048) > 0  # 2x the blocks: larger maps
    for bad_b in (32, 96, 256):
        assert fp.fp_workspace_bytes(4, 1, 2048, block_size=bad_b) == 0
    assert fp.fp_col_idx_capacity(131072, 64) == 2048 * 2049 // 2
    assert fp.fp_workspace_bytes(4, 1, 100, block_size=64) == 0       # n < 128
    assert fp.fp_workspace_bytes(1, 1, (1 << 19) + 64, block_size=64) == 0  # nb > 8192
    assert fp.fp_workspace_bytes(1, 1, 1 << 19, block_size=64) > 0


def test_validation_codes_without_device(lib):
    ws_bytes = fp.fp_workspace_bytes(4, 1, 2048)
    P = 0x10000  # fake, 16-B aligned; never dereferenced by validation
    L = lib
    s = ctypes.c_void_p(0)
    assert L.fp_plan(None, P, 4, 1, 2048, 128, 128, 0.1, P, ws_bytes, P, P, s) == 1
    assert L.fp_plan(P, P, 4, 3, 2048, 128, 128, 0.1, P, ws_bytes, P, P, s) == 2
    assert L.fp_plan(P, P, 4, 1, 127, 128, 128, 0.1, P, ws_bytes, P, P, s) == 2
    assert L.fp_plan(P, P, 4, 1, (1 << 20) + 128, 128, 128, 0.1, P, ws_bytes, P, P, s) == 2
    assert L.fp_plan(P, P, 4, 1, 2048, 64, 128, 0.1, P, ws_bytes, P, P, s) == 2
    assert L.fp_plan(P, P, 4, 1, 2048, 128, 128, -0.1, P, ws_bytes, P, P, s) == 3
    assert L.fp_plan(P, P, 4, 1, 2048, 128, 128, float("nan"), P, ws_bytes, P, P, s) == 3
    assert L.fp_plan(P + 8, P, 4, 1, 2048, 128, 128, 0.1, P, ws_bytes, P, P, s) == 4
    assert L.fp_plan(P, P, 4, 1, 2048, 128, 128, 0.1, P, ws_bytes - 1, P, P, s) == 5
    assert L.fp_select(4, 1, 2048, 128, 128, 0.0, 0, P, ws_bytes, P, P, None, s) == 3
    assert L.fp_select(4, 1, 2048, 128, 128, 0.9, -1, P, ws_bytes, P, P, None, s) == 3
    assert L.fp_select(4, 1, 2048, 128, 128, float("nan"), 0, P, ws_bytes, P, P, None, s) == 3
    assert L.fp_select(4, 1, 2048, 128, 128, 0.9, 0, P, ws_bytes, None, P, None, s) == 1
    assert L.fp_sparse_attn(P, P, P, P, 4, 1, 2048, 128, 128, None, P, P, ws_bytes, s) == 1
    assert L.fp_sparse_attn(P, P, P, P + 4, 4, 1, 2048, 128, 128, P, P, P, ws_bytes, s) == 4
    # all arguments valid: on a box without an sm_100 device -> FP_ERR_DEVICE
    import torch
    if not torch.cuda.is_available():
        assert L.fp_plan(P, P, 4, 1, 2048, 128, 128, 0.1, P, ws_bytes, P, P, s) == 6
        assert L.fp_dense_causal_attn(P, P, P, P, 4, 1, 2048, 128, 128, None, 0, s) == 6
    for code in range(8):
        assert L.fp_status_string(code)


def test_binding_raises_without_fallback(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(Exception):
        fp.FlexPrefill(4, 1, 2048)


def test_select_ex_option_validation(lib):
    ws_bytes = fp.fp_workspace_bytes(4, 1, 2048)
    P = 0x10000
    s = ctypes.c_void_p(0)
    for bad in [(2, 0, 0), (0, -1, 0), (0, 0, -128)]:
        opt = fp.SelectOptions(*bad)
        assert lib.fp_select_ex(4, 1, 2048, 128, 128, 0.9, 0, ctypes.byref(opt), P, ws_bytes, P, P,
                                None, s) == 3, bad
    # a maximum budget below the minimum budget would undercut the per-row floor (A23)
    opt = fp.SelectOptions(0, 0, 1024)
    assert lib.fp_select_ex(4, 1, 2048, 128, 128, 0.9, 2048, ctypes.byref(opt), P, ws_bytes, P, P,
                            None, s) == 3
    import torch
    if not torch.cuda.is_available():  # valid options -> device check
        assert lib.fp_select_ex(4, 1, 2048, 128, 128, 0.9, 1024, ctypes.byref(opt), P, ws_bytes, P,
                                P, None, s) == 6
        # budgets near INT_MAX: converted in 64-bit arithmetic, no overflow
        big = fp.SelectOptions(0, 0, 2**31 - 1)
        assert lib.fp_select_ex(4, 1, 2048, 128, 128, 0.9, 2**31 - 2, ctypes.byref(big), P,
                                ws_bytes, P, P, None, s) == 6
        opt = fp.SelectOptions(1, 1, 4096)
        assert lib.fp_select_ex(4, 1, 2048, 128, 128, 0.9, 0, ctypes.byref(opt), P, ws_bytes, P, P,
                                None, s) == 6
        assert lib.fp_select_ex(4, 1, 2048, 128, 128, 0.9, 0, None, P, ws_bytes, P, P, None, s) == 6


def test_ragged_sizes(lib):
    # ragged n (A26): nb = ceil(n / 128); capacity and workspace grow accordingly
    assert fp.fp_col_idx_capacity(2085) == 17 * 18 // 2
    assert fp.fp_col_idx_capacity(129) == 3
    assert fp.fp_workspace_bytes(4, 1, 2085) > fp.fp_workspace_bytes(4, 1, 2048)
    assert fp.fp_workspace_bytes(4, 1, 129) > 0


def test_layout_helpers_and_validation(lib):
    n, H, G = 1000, 8, 2
    a = fp.fp_layout_bhsd(3, H, G, n)
    assert a.batch == 3
    assert list(a.q_stride) == [H * n * 128, n * 128, 128] == list(a.o_stride)
    assert list(a.k_stride) == [G * n * 128, n * 128, 128] == list(a.v_stride)
    b = fp.fp_layout_bshd(2, H, G, n)
    assert list(b.q_stride) == [n * H * 128, 128, H * 128]
    assert list(b.k_stride) == [n * G * 128, 128, G * 128]
    with pytest.raises(fp.FlexPrefillError):
        fp.fp_layout_bshd(0, H, G, n)
    P = 0x10000
    s = ctypes.c_void_p(0)
    ws_bytes = fp.fp_workspace_bytes(2 * H, 2 * G, n)
    L = lib
    bad = fp.fp_layout_bshd(2, H, G, n)
    bad.k_stride[2] = 1004  # not a multiple of 8 elements
    assert L.fp_plan_ex(P, P, H, G, n, 128, 128, ctypes.byref(bad), 0.1, P, ws_bytes, P, P, s) == 4
    bad = fp.fp_layout_bshd(2, H, G, n)
    bad.q_stride[1] = 64  # rows / heads closer than 128 elements
    assert L.fp_plan_ex(P, P, H, G, n, 128, 128, ctypes.byref(bad), 0.1, P, ws_bytes, P, P, s) == 2
    bad = fp.fp_layout_bshd(2, H, G, n)
    bad.batch = 0
    assert L.fp_sparse_attn_ex(P, P, P, P, H, G, n, 128, 128, ctypes.byref(bad), P, P, P, 0, s) == 2
    ok = fp.fp_layout_bshd(2, H, G, n)
    # the workspace covers batch * heads flattened heads
    assert L.fp_plan_ex(P, P, H, G, n, 128, 128, ctypes.byref(ok), 0.1, P,
                        fp.fp_workspace_bytes(H, G, n), P, P, s) == 5
    import torch
    if not torch.cuda.is_available():
        assert L.fp_plan_ex(P, P, H, G, n, 128, 128, ctypes.byref(ok), 0.1, P, ws_bytes, P, P, s) == 6
        assert L.fp_plan_ex(P, P, H, G, n, 128, 128, None, 0.1, P, ws_bytes, P, P, s) == 6
        assert L.fp_dense_causal_attn_ex(P, P, P, P, H, G, n, 128, 128, ctypes.byref(ok), None, 0,
                                         s) == 6


def test_peers_validation(lib):
    """fp_sparse_attn_peers (next row f4): argument checks before any device work."""
    P = 0x10000
    s = ctypes.c_void_p(0)
    H, G, n = 4, 1, 2048
    L = lib
    f = L.fp_sparse_attn_peers
    assert f(P, P, P, P, P, 9, H, G, n, 128, 128, None, P, P, P, 0, s) == 3   # n_peer > FP_MAX_PEERS
    assert f(P, P, P, P, P, -1, H, G, n, 128, 128, None, P, P, P, 0, s) == 3
    assert f(P, P, P, P, None, 2, H, G, n, 128, 128, None, P, P, P, 0, s) == 1  # peer_o NULL
    assert f(P, P, P, P, P + 4, 2, H, G, n, 128, 128, None, P, P, P, 0, s) == 4  # peer_o not 8-B aligned
    assert f(P, P, P, P, P, 2, H, G, n, 128, 128, None, None, P, P, 0, s) == 1  # CSR NULL
    assert f(P, P, P, P, P, 2, H, 3, n, 128, 128, None, P, P, P, 0, s) == 2
    import torch
    # ws is optional scheduler scratch: non-NULL must be a full workspace
    assert f(P, P, P, P, P, 2, H, G, n, 128, 128, None, P, P, P, 0, s) == 5
    assert f(P, P, P, P, P, 2, H, G, n, 128, 128, None, P, P, P + 8, 1 << 40, s) == 4
    if not torch.cuda.is_available():
        assert f(P, P, P, P, P, 2, H, G, n, 128, 128, None, P, P, None, 0, s) == 6
        assert f(P, P, P, P, None, 0, H, G, n, 128, 128, None, P, P, None, 0, s) == 6
        ws_bytes = fp.fp_workspace_bytes(H, G, n)
        assert f(P, P, P, P, None, 0, H, G, n, 128, 128, None, P, P, P, ws_bytes, s) == 6


def test_layer_host_validates_everything_first(lib):
    """fp_layer_host checks every argument of its nested calls before the first
    copy is enqueued (an invalid call enqueues nothing)."""
    H, G, n = 8, 2, 2048
    ws_bytes = fp.fp_workspace_bytes(H, G, n)
    P = 0x10000
    s = ctypes.c_void_p(0)
    f = lib.fp_layer_host

    def call(**kw):
        a = dict(qh=P, kh=P, vh=P, oh=P, dq=P, dk=P, dv=P, do=P, H=H, G=G, n=n, d=128, b=128,
                 gamma=0.9, tau=0.1, mb=0, ws=P, wsb=ws_bytes, pat=P, jsd=P, rp=P, ci=P)
        a.update(kw)
        return f(a["qh"], a["kh"], a["vh"], a["oh"], a["dq"], a["dk"], a["dv"], a["do"], a["H"],
                 a["G"], a["n"], a["d"], a["b"], a["gamma"], a["tau"], a["mb"], a["ws"], a["wsb"],
                 a["pat"], a["jsd"], a["rp"], a["ci"], s)
    assert call(oh=None) == 1
    assert call(ci=None) == 1
    assert call(G=3) == 2
    assert call(gamma=0.0) == 3
    assert call(tau=1.5) == 3
    assert call(mb=-1) == 3
    assert call(do=P + 8) == 4     # device output not 16-B aligned
    assert call(ws=P + 4) == 4
    assert call(rp=P + 2) == 4     # int32 arrays need 4-B alignment
    assert call(wsb=ws_bytes - 1) == 5
    import torch
    if not torch.cuda.is_available():
        assert call() == 6
