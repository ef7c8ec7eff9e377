// fp_attn9.cu -- stage (iii) of FlexPrefill, y = A(Q, K, V, S) (P:66-83,
// P:287-288), version 9: v5's single-stream tile pipeline run over the key
// blocks of a q-block PAIR, so each K/V tile fetched from L2 serves both rows.
//
// v5 (fp_attn.cu) loads 64 KiB of K/V per computed (q-block, k-block) tile;
// v8 (fp_attn8.cu) shares those loads between rows qb and qb-1 (0.59 loads per
// tile at C3, tools/pair_study.py) but splits the softmax into two one-warp-
// per-scheduler warpgroups whose S/P buffers serialise with their own P.V.
// Here the pair's work is ONE stream of ops: for each entry e of the union of
// the two sorted CSR rows, an op for row A (= qbA) if A selected e, then one
// for row B (= qbA - 1) if B did. Every op is processed exactly like a v5
// tile: S_k = Q_x K_e^T into TMEM buffer k & 1 (issued two ops ahead), all 8
// softmax warps on it (16x256b TMEM shape, quad-shuffle row reductions, lazy
// running max), P over S, O_x += P_k V_e. Rows A and B have their own O
// accumulator and (max, sum) state.
//
// One CTA per (head, q-block pair) work item, 384 threads:
//   warp 8   K producer   Q_A, Q_B, then the K tiles of the union entries (2-stage ring)
//   warp 10  V producer   V tiles of the union entries (3-stage ring)
//   warp 9   MMA issuer   S (both operands in smem, Q_x K-major) and P.V (P in TMEM)
//   warps 0-7 softmax     as v5, state of the op's row
// TMEM (512 columns): S/P buffers [0,128) [128,256), O_A [256,384), O_B [384,512).
// Each row's diagonal block (kb == qb_x) takes the intra-block causal mask.
#include <math.h>

#include "fp_common.cuh"
#include "fp_internal.h"

namespace fp {

namespace {

constexpr int kThreads9 = 384;
constexpr int kKS9 = 2, kVS9 = 3;  // K / V ring depths (tiles)
constexpr uint32_t kColO9 = 256;
constexpr float kRescale9 = 8.0f;  // lazy rescale: tolerate P up to 2^8 (as v5)

struct Attn9Smem {
  uint8_t q[2][kTileBytes];  // Q_A, Q_B (1024-B aligned: first member)
  uint8_t k[kKS9][kTileBytes];
  uint8_t v[kVS9][kTileBytes];
  uint64_t q_full;
  uint64_t k_full[kKS9], k_empty[kKS9];
  uint64_t v_full[kVS9], v_empty[kVS9];
  uint64_t s_full[2], p_full[2];  // per S/P buffer
  uint64_t pv_done[2];            // per row (A, B)
  uint32_t tmem_base;
};

FP_DEV float fmax3_9(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
FP_DEV void ffma2_9(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0, float c1) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
FP_DEV void fadd2_9(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
FP_DEV float quad_max9(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
FP_DEV float quad_sum9(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v + __shfl_xor_sync(0xffffffffu, v, 2);
}

// S = Q K^T, M=128 N=128, 8 k-steps in one asm statement; both operands
// K-major SW128 tiles of two 16 KiB boxes (k-step kk: box kk/4, byte (kk%4)*32).
FP_DEV void umma_ss_chain8_9(uint32_t d, uint64_t a0, uint64_t b0, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %9, %17, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %10, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %11, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %12, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %5, %13, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %6, %14, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %7, %15, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %8, %16, %17, p;\n\t}" ::"r"(d),
      "l"(a0), "l"(a0 + 2), "l"(a0 + 4), "l"(a0 + 6), "l"(a0 + 1024), "l"(a0 + 1026),
      "l"(a0 + 1028), "l"(a0 + 1030), "l"(b0), "l"(b0 + 2), "l"(b0 + 4), "l"(b0 + 6),
      "l"(b0 + 1024), "l"(b0 + 1026), "l"(b0 + 1028), "l"(b0 + 1030), "r"(idesc));
}
// O += P V, 8 k-steps (16 keys each): A = P in TMEM columns a0 + 8 kk, B = V
// (MN-major SW128) descriptor b0 + kk * 2048 B.
FP_DEV void umma_pv_chain8_9(uint32_t d, uint32_t a0, uint64_t b0, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, 1, 0;\n\tsetp.ne.b32 q, %18, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %9, %17, q;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %10, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%3], %11, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%4], %12, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%5], %13, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%6], %14, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%7], %15, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], %16, %17, p;\n\t}" ::"r"(d),
      "r"(a0), "r"(a0 + 8), "r"(a0 + 16), "r"(a0 + 24), "r"(a0 + 32), "r"(a0 + 40), "r"(a0 + 48),
      "r"(a0 + 56), "l"(b0), "l"(b0 + 128), "l"(b0 + 256), "l"(b0 + 384), "l"(b0 + 512),
      "l"(b0 + 640), "l"(b0 + 768), "l"(b0 + 896), "r"(idesc), "r"(acc0));
}

// The pair's op stream: entries of the union of the two sorted CSR rows; per
// entry an op for row A (if selected), then one for row B (if selected).
struct PairOps {
  const int32_t* la;
  const int32_t* lb;
  int na, nb_, ia, ib;
  int e, mask, kb;  // current entry, its not-yet-emitted rows, its key block
  bool dense;
  FP_DEV bool done() const { return mask == 0 && ia >= na && ib >= nb_; }
  // next op: returns its row x (0 = A, 1 = B); e_out = union entry, kb_out =
  // key block, last = the entry's last op
  FP_DEV int next(int& e_out, int& kb_out, bool& last) {
    if (mask == 0) {
      const int ka = ia < na ? (dense ? ia : __ldg(la + ia)) : 0x7fffffff;
      const int kbb = ib < nb_ ? (dense ? ib : __ldg(lb + ib)) : 0x7fffffff;
      kb = min(ka, kbb);
      mask = (ka == kb ? 1 : 0) | (kbb == kb ? 2 : 0);
      ia += mask & 1;
      ib += mask >> 1;
      ++e;
    }
    const int x = (mask & 1) ? 0 : 1;
    mask &= ~(1 << x);
    e_out = e;
    kb_out = kb;
    last = (mask == 0);
    return x;
  }
};

// One key tile for one softmax thread (v5's): rows R0 and R0 + 8 of its 16-lane
// group, columns 8k + 2a, 8k + 2a + 1 (16x256b register order).
template <bool DIAG>
FP_DEV void softmax_tile9(float* v, int R0, int a, float scale_log2, float* m_used, float* alpha,
                          float* rs) {
  if (DIAG) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int c0 = 8 * k + 2 * a;
      if (c0 > R0) v[4 * k] = -INFINITY;
      if (c0 + 1 > R0) v[4 * k + 1] = -INFINITY;
      if (c0 > R0 + 8) v[4 * k + 2] = -INFINITY;
      if (c0 + 1 > R0 + 8) v[4 * k + 3] = -INFINITY;
    }
  }
  float p0 = fmax3_9(v[0], v[1], v[4]), p1 = fmax3_9(v[5], v[8], v[9]);
  float q0 = fmax3_9(v[2], v[3], v[6]), q1 = fmax3_9(v[7], v[10], v[11]);
#pragma unroll
  for (int k = 3; k < 16; k += 2) {
    p0 = fmax3_9(p0, v[4 * k], v[4 * k + 1]);
    q0 = fmax3_9(q0, v[4 * k + 2], v[4 * k + 3]);
    if (k + 1 < 16) {
      p1 = fmax3_9(p1, v[4 * k + 4], v[4 * k + 5]);
      q1 = fmax3_9(q1, v[4 * k + 6], v[4 * k + 7]);
    }
  }
  const float mx0 = quad_max9(fmaxf(p0, p1)) * scale_log2;
  const float mx1 = quad_max9(fmaxf(q0, q1)) * scale_log2;
  alpha[0] = 1.f;
  alpha[1] = 1.f;
  if (mx0 > m_used[0] + kRescale9) {
    alpha[0] = exp2f(m_used[0] - mx0);  // 0 on the row's first tile
    m_used[0] = mx0;
  }
  if (mx1 > m_used[1] + kRescale9) {
    alpha[1] = exp2f(m_used[1] - mx1);
    m_used[1] = mx1;
  }
  const float n0 = -m_used[0], n1 = -m_used[1];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    ffma2_9(v[4 * k], v[4 * k + 1], v[4 * k], v[4 * k + 1], scale_log2, scale_log2, n0, n0);
    ffma2_9(v[4 * k + 2], v[4 * k + 3], v[4 * k + 2], v[4 * k + 3], scale_log2, scale_log2, n1, n1);
  }
#pragma unroll
  for (int k = 0; k < 64; ++k) v[k] = fast_exp2(v[k]);
  float s0 = 0.f, s1 = 0.f, t0 = 0.f, t1 = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    fadd2_9(s0, s1, s0, s1, v[4 * k], v[4 * k + 1]);
    fadd2_9(t0, t1, t0, t1, v[4 * k + 2], v[4 * k + 3]);
  }
  rs[0] = s0 + s1;
  rs[1] = t0 + t1;
}

template <bool DENSE>
__global__ void __launch_bounds__(kThreads9, 1)
    attn9_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                 const __grid_constant__ CUtensorMap vmap, __nv_bfloat16* __restrict__ o,
                 const TLayout ol, int Hp, int Gp, int H, int G, int n, int nb, long long cap,
                 const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                 float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (smem_u32(smem_raw) & 1023u) __trap();  // SW128 tiles need 1024-B alignment
  Attn9Smem& sm = *reinterpret_cast<Attn9Smem*>(smem_raw);

  const int tid = threadIdx.x;
  const int wid = warp_id();
  // work item (KV-group-major, q-block pairs descending, heads of the group interleaved)
  const int gsz = H / G;
  const int npair = (nb + 1) >> 1;
  const int per_group = gsz * npair;
  const int g = blockIdx.x / per_group;
  const int rem = blockIdx.x - g * per_group;
  const int qbA = nb - 1 - 2 * (rem / gsz);
  const int qbB = qbA - 1;  // -1: no row B
  const int h = g * gsz + rem % gsz;
  int nA, nB;
  const int32_t* la = nullptr;
  const int32_t* lb = nullptr;
  if (DENSE) {
    nA = qbA + 1;
    nB = qbB + 1;
  } else {
    const int32_t* rp = row_ptr + (size_t)h * (nb + 1);
    const int bA = rp[qbA];
    nA = rp[qbA + 1] - bA;
    la = col_idx + (size_t)h * cap + bA;
    if (qbB >= 0) {
      const int bB = rp[qbB];
      nB = bA - bB;
      lb = col_idx + (size_t)h * cap + bB;
    } else {
      nB = 0;
    }
  }

  if (wid == 9) tmem_alloc(&sm.tmem_base, 512);
  if (tid == 256) {
    tma_prefetch_desc(&qmap);
    tma_prefetch_desc(&kmap);
    tma_prefetch_desc(&vmap);
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < kKS9; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < kVS9; ++s) {
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.s_full[b], 1);
      mbar_init(&sm.p_full[b], 256);
      mbar_init(&sm.pv_done[b], 1);
    }
    mbar_fence_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm.tmem_base;

  if (wid >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
    if (wid == 8 || wid == 10) {
      // ------------------------------------------------ TMA producers (K: warp 8, V: warp 10)
      if (lane_id() == 0) {
        const bool isK = (wid == 8);
        const uint64_t pol = policy_evict_last();
        if (isK) {
          mbar_arrive_expect_tx(&sm.q_full, nB > 0 ? 2 * kTileBytes : kTileBytes);
          tma_tile(sm.q[0], &qmap, &sm.q_full, qbA * 128, h, Hp);
          if (nB > 0) tma_tile(sm.q[1], &qmap, &sm.q_full, qbB * 128, h, Hp);
        }
        const int depth = isK ? kKS9 : kVS9;
        uint64_t* full = isK ? sm.k_full : sm.v_full;
        uint64_t* empty = isK ? sm.k_empty : sm.v_empty;
        const CUtensorMap* map = isK ? &kmap : &vmap;
        PairOps ops{la, lb, nA, nB, 0, 0, -1, 0, 0, DENSE};
        int ne = 0;
        while (!ops.done()) {
          int e, kb;
          bool last;
          ops.next(e, kb, last);
          if (!last) continue;  // one load per union entry
          const int s = e % depth;
          if (e >= depth) mbar_wait(&empty[s], ((e - depth) / depth) & 1);
          mbar_arrive_expect_tx(&full[s], kTileBytes);
          tma_tile_hint(isK ? sm.k[s] : sm.v[s], map, &full[s], kb * 128, g, Gp, pol);
          ne = e + 1;
        }
        // drain: the issuer releases every entry's slot; consume those
        // releases before the CTA exits
        for (int d = max(0, ne - depth); d < ne; ++d) mbar_wait(&empty[d % depth], (d / depth) & 1);
      }
    } else if (wid == 9) {
      // ------------------------------------------------ MMA issuer
      if (lane_id() == 0) {
        constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false);
        constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, true);
        const uint64_t qdesc0 = sdesc_kmajor(smem_u32(sm.q[0]), 0);
        const uint64_t qdesc1 = sdesc_kmajor(smem_u32(sm.q[1]), 0);
        PairOps ops{la, lb, nA, nB, 0, 0, -1, 0, 0, DENSE};
        int nops = 0;  // ops whose S has been issued
        // issue S for the next op; returns its (row, union entry, last-of-entry)
        auto issue_s = [&](int& x, int& e, bool& last) {
          int kb;
          x = ops.next(e, kb, last);
          const int ks = e % kKS9;
          mbar_wait(&sm.k_full[ks], (e / kKS9) & 1);
          tc_fence_after();
          const int b = nops & 1;
          umma_ss_chain8_9(tbase + b * 128, x ? qdesc1 : qdesc0, sdesc_kmajor(smem_u32(sm.k[ks]), 0),
                           idesc_s);
          umma_commit(&sm.s_full[b]);
          if (last) umma_commit(&sm.k_empty[ks]);
          ++nops;
        };
        // ops k (x0), k + 1 (x1) in flight; S is issued two ops ahead
        int x0 = 0, e0 = 0, x1 = 0, e1 = 0, x2 = 0, e2 = 0;
        bool l0 = false, l1 = false, l2 = false;
        mbar_wait(&sm.q_full, 0);
        issue_s(x0, e0, l0);
        if (!ops.done()) issue_s(x1, e1, l1);
        int pv_a = 0, pv_b = 0;
        for (int k = 0; k < nops; ++k) {
          const int vs = e0 % kVS9;
          mbar_wait(&sm.v_full[vs], (e0 / kVS9) & 1);
          mbar_wait(&sm.p_full[k & 1], (k >> 1) & 1);
          tc_fence_after();
          umma_pv_chain8_9(tbase + kColO9 + x0 * 128, tbase + (k & 1) * 128,
                           sdesc_mnmajor(smem_u32(sm.v[vs]), 0), idesc_o, x0 ? pv_b > 0 : pv_a > 0);
          if (x0) ++pv_b; else ++pv_a;
          if (l0) umma_commit(&sm.v_empty[vs]);
          umma_commit(&sm.pv_done[x0]);
          if (!ops.done()) issue_s(x2, e2, l2);
          x0 = x1; e0 = e1; l0 = l1;
          x1 = x2; e1 = e2; l1 = l2;
        }
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;");
    // ------------------------------------------------ softmax warps 0-7 (v5 layout)
    // warp w: TMEM lanes (w & 3) * 32 + (w >> 2) * 16 .. +16; thread: rows
    // R0 = base + lane / 4 and R0 + 8, columns 8k + 2a, 8k + 2a + 1 (a = lane % 4)
    const int lbase = (wid & 3) * 32 + (wid >> 2) * 16;
    const int a = lane_id() & 3;
    const int R0 = lbase + (lane_id() >> 2);
    const uint32_t lane_off = (uint32_t)lbase << 16;
    // state of the current op's row and of the other row (swapped on a change)
    int cx = 0;
    float m_c[2] = {-INFINITY, -INFINITY}, l_c[2] = {0.f, 0.f};
    float m_o[2] = {-INFINITY, -INFINITY}, l_o[2] = {0.f, 0.f};
    int cnt_c = 0, cnt_o = 0;  // ops processed per row
    PairOps ops{la, lb, nA, nB, 0, 0, -1, 0, 0, DENSE};
    for (int k = 0; !ops.done(); ++k) {
      int e, kb;
      bool last;
      const int x = ops.next(e, kb, last);
      if (x != cx) {
        cx = x;
        float t;
        t = m_c[0]; m_c[0] = m_o[0]; m_o[0] = t;
        t = m_c[1]; m_c[1] = m_o[1]; m_o[1] = t;
        t = l_c[0]; l_c[0] = l_o[0]; l_o[0] = t;
        t = l_c[1]; l_c[1] = l_o[1]; l_o[1] = t;
        const int ti = cnt_c; cnt_c = cnt_o; cnt_o = ti;
      }
      const int b = k & 1;
      const uint32_t tS = tbase + b * 128 + lane_off;
      const uint32_t tO = tbase + kColO9 + x * 128 + lane_off;
      mbar_wait(&sm.s_full[b], (k >> 1) & 1);
      tc_fence_after();
      float v[64];
      tmem_ld_16x256b_x16(tS, reinterpret_cast<uint32_t*>(v));
      tmem_wait_ld();
      float alpha[2], rs[2];
      if (kb == (x ? qbB : qbA))  // the row's diagonal block (its last)
        softmax_tile9<true>(v, R0, a, scale_log2, m_c, alpha, rs);
      else
        softmax_tile9<false>(v, R0, a, scale_log2, m_c, alpha, rs);
      l_c[0] = l_c[0] * alpha[0] + rs[0];
      l_c[1] = l_c[1] * alpha[1] + rs[1];
      // every PV completion of this row is consumed (normally long complete):
      // O_x then holds the row's earlier P V and may be rescaled
      if (cnt_c > 0) {
        mbar_wait(&sm.pv_done[x], (cnt_c - 1) & 1);
        if (__any_sync(0xffffffffu, alpha[0] != 1.f || alpha[1] != 1.f)) {
          tc_fence_after();
          float ov[64];
          tmem_ld_16x256b_x16(tO, reinterpret_cast<uint32_t*>(ov));
          tmem_wait_ld();
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            ov[4 * j] *= alpha[0];
            ov[4 * j + 1] *= alpha[0];
            ov[4 * j + 2] *= alpha[1];
            ov[4 * j + 3] *= alpha[1];
          }
          tmem_st_16x256b_x16(tO, reinterpret_cast<uint32_t*>(ov));
        }
      }
      ++cnt_c;
      // P (bf16 pairs): packed column 4j + a holds keys 8j + 2a, 8j + 2a + 1
      uint32_t pk[32];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        pk[2 * j] = pack_bf16x2(v[4 * j], v[4 * j + 1]);
        pk[2 * j + 1] = pack_bf16x2(v[4 * j + 2], v[4 * j + 3]);
      }
      tmem_st_16x128b_x16(tS, pk);
      tmem_wait_st();
      tc_fence_before();
      mbar_arrive(&sm.p_full[b]);
    }
    // epilogue, per row: O / l -> bf16 -> global (rows past n are not stored)
#pragma unroll 1
    for (int x = 0; x < 2; ++x) {
      const int cnt = (x == cx) ? cnt_c : cnt_o;
      if (cnt == 0) continue;
      const float* lx = (x == cx) ? l_c : l_o;
      const float il0 = 1.0f / quad_sum9(lx[0]), il1 = 1.0f / quad_sum9(lx[1]);
      mbar_wait(&sm.pv_done[x], (cnt - 1) & 1);
      tc_fence_after();
      float ov[64];
      tmem_ld_16x256b_x16(tbase + kColO9 + x * 128 + lane_off, reinterpret_cast<uint32_t*>(ov));
      tmem_wait_ld();
      const int row0 = (x ? qbB : qbA) * 128 + R0;
      uint32_t* d0 = reinterpret_cast<uint32_t*>(o + toff(ol, h, row0)) + a;
      uint32_t* d1 = d0 + 4 * ol.rs;  // row R0 + 8
      if (row0 < n) {
#pragma unroll
        for (int j = 0; j < 16; ++j) d0[4 * j] = pack_bf16x2(ov[4 * j] * il0, ov[4 * j + 1] * il0);
      }
      if (row0 + 8 < n) {
#pragma unroll
        for (int j = 0; j < 16; ++j) d1[4 * j] = pack_bf16x2(ov[4 * j + 2] * il1, ov[4 * j + 3] * il1);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 9) tmem_dealloc(tbase, 512);
}

}  // namespace

size_t attn9_smem_bytes() { return sizeof(Attn9Smem); }

cudaError_t launch_attn_v9(const Shape& s, const Layout& lay, const CUtensorMap& qmap,
                           const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                           const int32_t* row_ptr, const int32_t* col_idx, bool dense,
                           cudaStream_t st) {
  static bool attr_done = false;
  const size_t smem = attn9_smem_bytes();
  if (!attr_done) {
    cudaFuncSetAttribute(attn9_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(attn9_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_done = true;
  }
  const float scale_log2 = (1.0f / sqrtf(128.0f)) * kLog2e;
  const dim3 grid(s.H * ((s.nb + 1) / 2));
  auto* op = reinterpret_cast<__nv_bfloat16*>(o);
  if (dense)
    attn9_kernel<true><<<grid, kThreads9, smem, st>>>(qmap, kmap, vmap, op, lay.o, lay.q.per,
                                                      lay.k.per, s.H, s.G, s.n, s.nb, s.tri,
                                                      row_ptr, col_idx, scale_log2);
  else
    attn9_kernel<false><<<grid, kThreads9, smem, st>>>(qmap, kmap, vmap, op, lay.o, lay.q.per,
                                                       lay.k.per, s.H, s.G, s.n, s.nb, s.tri,
                                                       row_ptr, col_idx, scale_log2);
  return cudaGetLastError();
}

}  // namespace fp
