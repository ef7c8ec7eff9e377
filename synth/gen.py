"""Seeded synthetic Q/K/V with planted attention structure.

This module is shared by the tests, the oracle timing leg and bench.py. It
holds NONE of FlexPrefill's arithmetic: it only draws numbers and rounds them
to bf16. Both the CUDA path and the float64 oracle consume the same bf16 bits.

Structure is planted in logit space (a component contributes
q_c . k_c / sqrt(d) to the logit), mirroring the paper's two head families:

* Structured / Vertical-Slash heads: an attention
  sink (keys 0..3), a few heavy vertical columns, a local slash (rotary pairs
  peaking at offset 0), a far slash (rotary pairs with a per-KV-head phase
  shift o*), and a per-key-block "warmth" that concentrates the diffuse mass
  in a subset of key blocks (so the rasterised selection is neither empty nor
  dense).
* Diverse / Query-Aware heads: each query block attends to the key
  blocks that share its cluster id (one-hot cluster axis), so the pooled
  estimate matches the true block distribution; plus a weak sink.

Q head h is Query-Aware-type iff h % g == g - 1 (g = H/G), giving "most heads
are VS". Logit boosts grow with lambda_n = ln(n/2048) so the planted
mass is not swamped by the background as n grows (SURVEY.md §7 hard part 3).

Per-head generators are independent (default_rng([seed, H, G, n, role, h])),
so a rank can build only its own head slice.
"""
import math
import numpy as np

D = 128
# dimension map (the two local-slash Dirichlet kernels
# take the "local" and "far" ranges, the warmth axis sits at 69)
BG = slice(0, 64)
SINK = 64
VERT = slice(65, 69)
WARM = 69
LOCAL = slice(70, 86)
FAR = slice(86, 102)
CLUSTER = slice(102, 118)
N_CLUSTERS = 16

# logit boosts (before + lambda_n) and shape knobs; calibrated with
# tools/calibrate_gen.py (results recorded in DESIGN.md)
GAINS = dict(
    bg_std=0.6,       # background components: logit noise std ~0.25
    sink=7.0,         # + lambda_n, keys 0..3
    vert=6.0,         # + lambda_n, per heavy-hitter column
    n_vert=(16, 32),  # heavy hitters at n = 2048 ...
    vert_growth=0.5,  # ... times (n / 2048)^vert_growth
    vert_skew=2.0,    # column j = n u^vert_skew (early-biased)
    local=7.5,        # + lambda_n, peak of the two Dirichlet local kernels
    period1=2048.0,
    period2=3000.0,
    warm=1.0,         # block warmth logit bias = warm * z_kb, z ~ N(0, 1)
    warm_frac=0.15,   # warmest fraction of blocks carry no heavy hitter
    cluster=8.0,      # + lambda_n, Query-Aware cluster match
    qa_sink=2.0,      # weak sink of Query-Aware heads (no lambda_n)
    head_jitter=0.05,
    lam_coef=0.6,     # boosts grow by lam_coef * ln(n / 2048)
)

ROLE_Q, ROLE_K, ROLE_V, ROLE_KVMETA, ROLE_QMETA = 1, 2, 3, 4, 5


def bf16_bits(x):
    """float32 -> bf16 bit pattern (uint16), round-to-nearest-even (A17)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    rounding = ((u >> 16) & 1) + np.uint32(0x7FFF)
    return ((u + rounding) >> 16).astype(np.uint16)


def bits_to_f32(bits):
    """bf16 bit pattern -> exact float32 value."""
    return (bits.astype(np.uint32) << 16).view(np.float32)


def bits_to_f64(bits):
    return bits_to_f32(bits).astype(np.float64)


def is_qa_type(h, heads, kv_heads):
    g = heads // kv_heads
    return (h % g) == (g - 1)


K_AMP = 3.0  # key-side amplitude of every planted single-dim component


def _amp(boost):
    """query-side amplitude so that (q * K_AMP) / sqrt(D) == boost."""
    return max(boost, 0.0) * math.sqrt(D) / K_AMP


def _ramp(boost):
    """query-side amplitude per rotary pair (8 pairs of key amplitude K_AMP):
    peak logit = 8 * q * K_AMP / sqrt(D) == boost."""
    return max(boost, 0.0) * math.sqrt(D) / (8.0 * K_AMP)


def _rng(seed, H, G, n, role, idx):
    return np.random.default_rng([seed, H, G, n, role, idx])


def _lam(n, gains=GAINS):
    return gains["lam_coef"] * math.log(max(n, 2048) / 2048.0)


def kv_meta(seed, H, G, n, g, gains=GAINS):
    """Per-KV-head planted structure: vertical columns, far shift, warm blocks, clusters."""
    r = _rng(seed, H, G, n, ROLE_KVMETA, g)
    nb = -(-n // 128)  # ragged n: the last block is partial
    # heavy hitters grow with context: n_vert * (n/2048)^vert_growth
    scale = (max(n, 2048) / 2048.0) ** gains["vert_growth"]
    nv = int(r.integers(gains["n_vert"][0], gains["n_vert"][1] + 1) * scale)
    # heavy-hitter columns, skewed toward early positions (j ~ n u^vert_skew)
    # block warmth z ~ N(0,1) per key block (logit bias warm * z for VS heads);
    # the warmest warm_frac of blocks host no heavy hitters
    warm = r.standard_normal(nb)
    u = r.random(nv)
    verts = np.unique(np.clip((n * u ** gains["vert_skew"]).astype(np.int64), 4, n - 1))
    # heavy hitters live outside the warm blocks (the warmth is the diffuse part)
    cut = np.quantile(warm, 1.0 - gains["warm_frac"]) if nb > 1 else np.inf
    verts = verts[warm[verts // 128] < cut]
    clusters = r.integers(0, N_CLUSTERS, nb)
    return dict(verts=verts, warm=warm, clusters=clusters)


def _dirichlet(pos, amp, period):
    """8 rotary pairs at harmonics f = 1..8 of one period: the dot product of a
    query row and a key row is amp_q amp_k sum_f cos(2 pi f (i - j) / period),
    a Dirichlet kernel -- a narrow bump at i - j = 0 (mod period) with low
    side lobes (a local window whose aliases every `period` tokens are weak
    because the two local components use coprime-ish periods)."""
    f = np.arange(1, 9)
    ang = np.outer(pos, 2.0 * np.pi * f / period)
    out = np.empty((pos.shape[0], 16), np.float32)
    out[:, 0::2] = amp * np.cos(ang)
    out[:, 1::2] = amp * np.sin(ang)
    return out


def make_k(seed, H, G, n, g, gains=GAINS):
    meta = kv_meta(seed, H, G, n, g, gains)
    r = _rng(seed, H, G, n, ROLE_K, g)
    K = np.zeros((n, D), np.float32)
    K[:, BG] = r.normal(0.0, gains["bg_std"], (n, 64))
    K[0:4, SINK] = K_AMP
    for t, j in enumerate(meta["verts"]):
        K[j, 65 + (t % 4)] = K_AMP
    pos = np.arange(n, dtype=np.float64)
    K[:, LOCAL] = _dirichlet(pos, K_AMP, gains["period1"])
    K[:, FAR] = _dirichlet(pos, K_AMP, gains["period2"])
    K[:, WARM] = K_AMP * np.repeat(meta["warm"], 128)[:n]
    K[0:4, WARM] = 0.0
    kb = np.arange(n) // 128
    K[np.arange(n), 102 + meta["clusters"][kb]] = K_AMP
    return K


def make_v(seed, H, G, n, g):
    r = _rng(seed, H, G, n, ROLE_V, g)
    return r.standard_normal((n, D), dtype=np.float32)


MIX_W = (0.2, 0.45, 0.7, 1.0)  # vertical share of the mixed heads, by KV group (mod 4)


def is_mixed(h, heads, kv_heads):
    g = heads // kv_heads
    return g > 1 and h % g == 0


def make_q(seed, H, G, n, h, gains=GAINS, mixed=False):
    """Q rows of head h. mixed=True (the C5 tau sweep): the
    first head of every KV group is Query-Aware-type plus a vertical
    (heavy-hitter) component of relative weight MIX_W[group % 4], which spreads
    D_JS across the swept tau range."""
    lam = _lam(n, gains)
    r = _rng(seed, H, G, n, ROLE_Q, h)
    rm = _rng(seed, H, G, n, ROLE_QMETA, h)
    Q = np.zeros((n, D), np.float32)
    Q[:, BG] = r.normal(0.0, gains["bg_std"], (n, 64))
    pos = np.arange(n, dtype=np.float64)
    # per-head component multipliers so heads of a group differ
    mult = rm.uniform(1.0 - gains["head_jitter"], 1.0 + gains["head_jitter"], 8)
    mix = mixed and is_mixed(h, H, G)
    if is_qa_type(h, H, G) or mix:
        Q[:, SINK] = _amp(gains["qa_sink"]) * mult[0]
        nb = -(-n // 128)  # ragged n: the last block is partial
        lam_h = rm.integers(0, N_CLUSTERS, nb)
        qb = np.arange(n) // 128
        Q[np.arange(n), 102 + lam_h[qb]] = _amp(gains["cluster"] + lam) * mult[1]
        if mix:
            Q[:, VERT] = MIX_W[(h * G // H) % 4] * _amp(gains["vert"] + lam) * mult[2]
    else:
        Q[:, SINK] = _amp(gains["sink"] + lam) * mult[0]
        Q[:, VERT] = _amp(gains["vert"] + lam) * mult[1]
        Q[:, LOCAL] = _dirichlet(pos, 0.5 * _ramp(gains["local"] + lam) * mult[2], gains["period1"])
        Q[:, FAR] = _dirichlet(pos, 0.5 * _ramp(gains["local"] + lam) * mult[3], gains["period2"])
        Q[:, WARM] = _amp(gains["warm"]) * mult[4]
    return Q


def make_layer_bits(w, heads=None, gains=GAINS):
    """Build bf16 bit arrays for a workload (synth.configs.Workload).

    heads: optional iterable of Q-head indices to build (others left zero);
    the KV heads they need are built. Returns (q, k, v) uint16 arrays shaped
    [H][n][128], [G][n][128], [G][n][128].
    """
    H, G, n = w.heads, w.kv_heads, w.seq_len
    hs = range(H) if heads is None else sorted(set(heads))
    gs = sorted({h * G // H for h in hs})
    q = np.zeros((H, n, D), np.uint16)
    k = np.zeros((G, n, D), np.uint16)
    v = np.zeros((G, n, D), np.uint16)
    for h in hs:
        q[h] = bf16_bits(make_q(w.seed, H, G, n, h, gains, getattr(w, "mixed", False)))
    for g in gs:
        k[g] = bf16_bits(make_k(w.seed, H, G, n, g, gains))
        v[g] = bf16_bits(make_v(w.seed, H, G, n, g))
    return q, k, v


def planted(w, gains=GAINS):
    """Ground truth of the planted structure, per KV head (for construction tests)."""
    return [kv_meta(w.seed, w.heads, w.kv_heads, w.seq_len, g, gains) for g in range(w.kv_heads)]
