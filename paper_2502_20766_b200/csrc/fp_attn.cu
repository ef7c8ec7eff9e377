// fp_attn.cu -- stage (iii) of FlexPrefill: y = A(Q, K, V, S) (P:66-83,
// P:287-288): causal block-sparse attention over the selected (q-block,
// k-block) pairs with online softmax and GQA, on tcgen05 tensor cores.
//
// One CTA per (head, query block) work item, warp-specialised (384 threads;
// registers rebalanced with setmaxnreg: 200 per softmax thread, 56 otherwise):
//   warp 8   K producer    Q tile once, then the K tiles of the row's key blocks
//                          (indices from the CSR) into a 3-stage TMA ring
//   warp 10  V producer    the V tiles into their own 3-stage ring
//   warp 9   MMA issuer    S_i = Q K_i^T into one of 3 TMEM S/P buffers, issued
//                          two tiles ahead; O += P_i V_i with P_i read from TMEM
//                          (tcgen05 "TS" form, A operand in tensor memory)
//   warps 0-7 softmax      two warps per TMEM lane quarter, 16 query rows each;
//                          TMEM is read with the 16x256b shape, so a row's 128
//                          scores are spread over a quad of threads (32 each,
//                          2 rows per thread): row max / sum need only quad
//                          shuffles. Online softmax in the log2 domain with a
//                          lazy running max (O is rescaled in TMEM only when the
//                          max grows by more than 2^8); P (bf16) written back
//                          over S (16x128b shape); final O / l -> global. An
//                          optional polynomial exp2 on the FMA pipe (FP_EMU)
//                          is compiled in but off by default (see below).
// TMEM (512 columns): S/P buffers 0..2 (128 each), O (128).
// The diagonal block (always the last of a row's sorted list) gets the
// intra-block causal mask (j <= i) in a separate code path. The dense causal
// kernel is the same template with the implicit list kb = 0..qb.
// Work order is KV-group-major (the K/V of one group, 64 MiB at 128k, stays
// in L2 while its heads run), query blocks descending within a group.
#include <math.h>

#include "fp_common.cuh"
#include "fp_internal.h"

#ifdef FP_TIMING
__device__ unsigned long long g_attn_timing[16];
#define FP_TMARK(k) do { if (timing_on) { long long _t = clock64(); tacc[k] += _t - tlast; tlast = _t; } } while (0)
#else
#define FP_TMARK(k) do { } while (0)
#endif

namespace fp {

namespace {

constexpr int kAttnThreads = 384;      // 8 softmax warps, K producer (8), MMA (9), V producer (10), spare (11)
// Measured on B200 (tools/attn_timing.py): under the 1 kW power cap the FMA-pipe
// exp2 costs more than it saves (C3 128k attn: 35.4 ms at 0, 36.7 at 12, 37.5
// at 20, 38.1 at 28 emulated values per thread), so the default is 0.
#ifndef FP_EMU
#define FP_EMU 0
#endif
constexpr int kEmuK = FP_EMU / 4;      // of each thread's 16 column groups (4 values), this many
                                       // are exponentiated on the FMA pipe
// FP_QTMEM: copy the Q tile into TMEM once (tcgen05.cp) so S = Q K^T reads only
// K from shared memory; TMEM then holds 2 S/P buffers + O + Q, and S_(i+2)
// reuses buffer (i & 1) right after PV_i is issued (in-order tcgen05 stream).
#ifndef FP_QTMEM
#define FP_QTMEM 1
#endif
constexpr int kSBuf = FP_QTMEM ? 2 : 3;  // S/P buffers in TMEM
constexpr uint32_t kColO = FP_QTMEM ? 256 : 384, kColQ = 384;
constexpr int kKV = 3;                 // K and V ring depths
#ifndef FP_RT
#define FP_RT 8.0f
#endif
constexpr float kRescaleThresh = FP_RT; // lazy rescale: tolerate P up to 2^FP_RT

struct AttnSmem {
  uint8_t q[kTileBytes];
  uint8_t k[kKV][kTileBytes];
  uint8_t v[kKV][kTileBytes];
  uint64_t q_full;
  uint64_t k_full[kKV], k_empty[kKV];
  uint64_t v_full[kKV], v_empty[kKV];
  uint64_t s_full[kSBuf], p_full[kSBuf], pv_done[kSBuf];
  uint32_t tmem_base;
};

FP_DEV float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
// (d0, d1) = (a0, a1) * (b0, b1) + (c0, c1) on the paired FMA pipe (FFMA2)
FP_DEV void ffma2(float& d0, float& d1, float a0, float a1, float b0, float b1, float c0, float c1) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1), "f"(c0), "f"(c1));
}
FP_DEV void fadd2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
// 2^x for a pair on the FMA/ALU pipes: x = j + f (j = rint(x), |f| <= 1/2),
// 2^f by a degree-3 minimax polynomial (max rel. error 7.5e-5; P is rounded to
// bf16 afterwards, 2^-9), 2^j added into the exponent field. x is clamped at
// -125 (the result is then < 2^-124, i.e. 0 for the bf16 P and the row sum).
FP_DEV void exp2_emu2(float x0, float x1, float& y0, float& y1) {
  const float kMagic = 12582912.0f;  // 1.5 * 2^23: rounds to an integer in the low mantissa bits
  x0 = fmaxf(x0, -125.0f);
  x1 = fmaxf(x1, -125.0f);
  float t0, t1, j0, j1, f0, f1, p0, p1;
  fadd2(t0, t1, x0, x1, kMagic, kMagic);
  fadd2(j0, j1, t0, t1, -kMagic, -kMagic);
  fadd2(f0, f1, x0, x1, -j0, -j1);
  ffma2(p0, p1, f0, f1, 0.0551716626f, 0.0551716626f, 0.242611155f, 0.242611155f);
  ffma2(p0, p1, p0, p1, f0, f1, 0.69326099f, 0.69326099f);
  ffma2(p0, p1, p0, p1, f0, f1, 0.999928072f, 0.999928072f);
  y0 = __uint_as_float(__float_as_uint(t0) * 8388608u + __float_as_uint(p0));
  y1 = __uint_as_float(__float_as_uint(t1) * 8388608u + __float_as_uint(p1));
}

// 8 k-steps of one M=128 x N=128 MMA chain in one asm statement: A from TMEM
// columns a0 + 8 kk, B descriptors b0 + off(kk) (off in 16-B units, added to
// the start-address field), so the issuing thread does no descriptor math per
// k-step. acc0: accumulate flag of the first k-step.
template <uint32_t O1, uint32_t O2, uint32_t O3, uint32_t O4, uint32_t O5, uint32_t O6, uint32_t O7>
FP_DEV void umma_ts_chain8(uint32_t d, uint32_t a0, uint64_t b0, uint32_t idesc, uint32_t acc0) {
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
      "r"(a0 + 56), "l"(b0), "l"(b0 + O1), "l"(b0 + O2), "l"(b0 + O3), "l"(b0 + O4), "l"(b0 + O5),
      "l"(b0 + O6), "l"(b0 + O7), "r"(idesc), "r"(acc0));
}
// k-step offsets (16-B units): K-major SW128 tile of two 16 KiB boxes
// (kk/4 box, (kk%4)*32 B) and the MN-major V tile (+2048 B per step)
#define FP_KMAJ_OFFS 2, 4, 6, 1024, 1026, 1028, 1030
#define FP_MNMAJ_OFFS 128, 256, 384, 512, 640, 768, 896

// One key tile of one softmax warpgroup: S row (128 fp32) from TMEM -> lazy
// running max -> P = 2^(s - m) (bf16) written over the S columns. Returns the
// row sum of P; updates m_used and sets alpha (scale for the previous O / l).
FP_DEV float quad_max(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 1));
  return fmaxf(v, __shfl_xor_sync(0xffffffffu, v, 2));
}
FP_DEV float quad_sum(float v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  return v + __shfl_xor_sync(0xffffffffu, v, 2);
}

// One key tile for one softmax thread: rows R0 = c and R1 = c + 8 of its
// 16-lane group (c = lane / 4), columns 8k + 2a, 8k + 2a + 1 (a = lane % 4).
// v: the 64 scores (16x256b register order). Returns the partial row sums.
template <bool DIAG>
FP_DEV void softmax_tile(float* v, int R0, int a, float scale_log2, float* m_used, float* alpha,
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
  // partial row maxima (raw logits; scale > 0), then across the quad
  float p0 = fmax3(v[0], v[1], v[4]), p1 = fmax3(v[5], v[8], v[9]);
  float q0 = fmax3(v[2], v[3], v[6]), q1 = fmax3(v[7], v[10], v[11]);
#pragma unroll
  for (int k = 3; k < 16; k += 2) {
    p0 = fmax3(p0, v[4 * k], v[4 * k + 1]);
    q0 = fmax3(q0, v[4 * k + 2], v[4 * k + 3]);
    if (k + 1 < 16) {
      p1 = fmax3(p1, v[4 * k + 4], v[4 * k + 5]);
      q1 = fmax3(q1, v[4 * k + 6], v[4 * k + 7]);
    }
  }
  const float mx0 = quad_max(fmaxf(p0, p1)) * scale_log2;
  const float mx1 = quad_max(fmaxf(q0, q1)) * scale_log2;
  // lazy running max per row: move only when it grows by more than 2^kRescaleThresh
  alpha[0] = 1.f;
  alpha[1] = 1.f;
  if (mx0 > m_used[0] + kRescaleThresh) {
    alpha[0] = exp2f(m_used[0] - mx0);  // 0 on the first tile
    m_used[0] = mx0;
  }
  if (mx1 > m_used[1] + kRescaleThresh) {
    alpha[1] = exp2f(m_used[1] - mx1);
    m_used[1] = mx1;
  }
  const float n0 = -m_used[0], n1 = -m_used[1];
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    ffma2(v[4 * k], v[4 * k + 1], v[4 * k], v[4 * k + 1], scale_log2, scale_log2, n0, n0);
    ffma2(v[4 * k + 2], v[4 * k + 3], v[4 * k + 2], v[4 * k + 3], scale_log2, scale_log2, n1, n1);
  }
#pragma unroll
  for (int k = 0; k < 16 - kEmuK; ++k)
#pragma unroll
    for (int e = 0; e < 4; ++e) v[4 * k + e] = fast_exp2(v[4 * k + e]);
#pragma unroll
  for (int k = 16 - kEmuK; k < 16; ++k) {
    exp2_emu2(v[4 * k], v[4 * k + 1], v[4 * k], v[4 * k + 1]);
    exp2_emu2(v[4 * k + 2], v[4 * k + 3], v[4 * k + 2], v[4 * k + 3]);
  }
  if (DIAG) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      const int c0 = 8 * k + 2 * a;
      if (c0 > R0) v[4 * k] = 0.f;
      if (c0 + 1 > R0) v[4 * k + 1] = 0.f;
      if (c0 > R0 + 8) v[4 * k + 2] = 0.f;
      if (c0 + 1 > R0 + 8) v[4 * k + 3] = 0.f;
    }
  }
  float s0 = 0.f, s1 = 0.f, t0 = 0.f, t1 = 0.f;
#pragma unroll
  for (int k = 0; k < 16; ++k) {
    fadd2(s0, s1, s0, s1, v[4 * k], v[4 * k + 1]);
    fadd2(t0, t1, t0, t1, v[4 * k + 2], v[4 * k + 3]);
  }
  rs[0] = s0 + s1;
  rs[1] = t0 + t1;
}

template <bool DENSE>
__global__ void __launch_bounds__(kAttnThreads, 1)
    attn_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                const __grid_constant__ CUtensorMap vmap, __nv_bfloat16* __restrict__ o,
                const TLayout ol, int Hp, int Gp, int H, int G, int n, int nb, long long cap,
                const int32_t* __restrict__ row_ptr,
                const int32_t* __restrict__ col_idx, float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // the 7 SW128 tiles fill 224 KiB: no room for alignment slack. The dynamic
  // shared memory window starts 1024-B aligned when the kernel has no static
  // shared memory; trap (fail loudly) if that ever stops holding.
  if (smem_u32(smem_raw) & 1023u) __trap();
  AttnSmem& sm = *reinterpret_cast<AttnSmem*>(smem_raw);

  const int tid = threadIdx.x;
  const int wid = warp_id();
  // work item (KV-group-major, q-blocks descending, heads of the group interleaved)
  const int gsz = H / G;
  const int per_group = gsz * nb;
  const int g = blockIdx.x / per_group;
  const int rem = blockIdx.x - g * per_group;
  const int qb = nb - 1 - rem / gsz;
  const int h = g * gsz + rem % gsz;
  int nk;
  const int32_t* list = nullptr;
  if (DENSE) {
    nk = qb + 1;
  } else {
    const int32_t* rp = row_ptr + (size_t)h * (nb + 1);
    const int beg = rp[qb];
    nk = rp[qb + 1] - beg;
    list = col_idx + (size_t)h * cap + beg;
  }

  if (wid == 9) tmem_alloc(&sm.tmem_base, 512);
  if (tid == 256) {  // warp 8 lane 0
    tma_prefetch_desc(&qmap);
    tma_prefetch_desc(&kmap);
    tma_prefetch_desc(&vmap);
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < kKV; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    for (int b = 0; b < kSBuf; ++b) {
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
  // producer / MMA warpgroup (warps 8-11) gives registers to the softmax warpgroups
  asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
  if (wid == 8 || wid == 10) {
    // ------------------------------------------------ TMA producers (K: warp 8, V: warp 10)
    if (lane_id() == 0) {
      const bool isK = (wid == 8);
      const uint64_t pol_kv = policy_evict_last();
      if (isK) {
        mbar_arrive_expect_tx(&sm.q_full, kTileBytes);
        tma_tile(sm.q, &qmap, &sm.q_full, qb * 128, h, Hp);
      }
      uint64_t* full = isK ? sm.k_full : sm.v_full;
      uint64_t* empty = isK ? sm.k_empty : sm.v_empty;
      const CUtensorMap* map = isK ? &kmap : &vmap;
      for (int i = 0; i < nk; ++i) {
        const int s = i % kKV;
        const int kb = DENSE ? i : __ldg(list + i);
        if (i >= kKV) mbar_wait(&empty[s], ((i - kKV) / kKV) & 1);
        mbar_arrive_expect_tx(&full[s], kTileBytes);
        tma_tile_hint(isK ? sm.k[s] : sm.v[s], map, &full[s], kb * 128, g, Gp, pol_kv);
      }
    }
  } else if (wid == 9) {
    // ------------------------------------------------ MMA issuer
    if (lane_id() == 0) {
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, true);
      const uint32_t qa = smem_u32(sm.q);
      auto issue_s = [&](int i) {
        const int s = i % kKV, b = i % kSBuf;
        mbar_wait(&sm.k_full[s], (i / kKV) & 1);
#if !FP_QTMEM
        // buffer b was last used by tile i-3: its P must have been consumed
        if (i >= kSBuf) mbar_wait(&sm.pv_done[b], ((i - kSBuf) / kSBuf) & 1);
#endif
        tc_fence_after();
        const uint32_t ka = smem_u32(sm.k[s]);
#if FP_QTMEM
        umma_ts_chain8<FP_KMAJ_OFFS>(tbase + b * 128, tbase + kColQ, sdesc_kmajor(ka, 0), idesc_s, 0);
#else
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)
          umma_bf16_ss(tbase + b * 128, sdesc_kmajor(qa, kk), sdesc_kmajor(ka, kk), idesc_s, kk > 0);
#endif
        umma_commit(&sm.s_full[b]);
        if (i + kKV < nk) umma_commit(&sm.k_empty[s]);  // the producer waits only for these
      };
      mbar_wait(&sm.q_full, 0);
#if FP_QTMEM
      tc_fence_after();
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)  // Q (K-major SW128 in smem) -> TMEM columns kColQ + 8 kk
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tbase + kColQ + kk * 8),
                     "l"(sdesc_kmajor(qa, kk)));
#endif
      issue_s(0);
      if (nk > 1) issue_s(1);
      for (int i = 0; i < nk; ++i) {
        const int s = i % kKV, b = i % kSBuf;
        mbar_wait(&sm.v_full[s], (i / kKV) & 1);
        mbar_wait(&sm.p_full[b], (i / kSBuf) & 1);
        tc_fence_after();
        const uint32_t va = smem_u32(sm.v[s]);
        umma_ts_chain8<FP_MNMAJ_OFFS>(tbase + kColO, tbase + b * 128, sdesc_mnmajor(va, 0), idesc_o,
                                      i > 0);
        umma_commit(&sm.pv_done[b]);
        if (i + kKV < nk) umma_commit(&sm.v_empty[s]);
        if (i + 2 < nk) issue_s(i + 2);
      }
    }
  }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;");
    // ------------------------------------------------ softmax warps 0-7
    // warp w: TMEM lanes (w & 3) * 32 + (w >> 2) * 16 .. +16; thread: rows
    // R0 = base + lane / 4 and R0 + 8, columns 8k + 2a, 8k + 2a + 1 (a = lane % 4)
    const int lbase = (wid & 3) * 32 + (wid >> 2) * 16;
    const int a = lane_id() & 3;
    const int R0 = lbase + (lane_id() >> 2);
    const uint32_t lane_off = (uint32_t)lbase << 16;
    const uint32_t tO = tbase + kColO + lane_off;
    float m_used[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};
#ifdef FP_TIMING
    const bool timing_on = (tid == 0);
    long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long tlast = clock64();
#endif
    for (int i = 0; i < nk; ++i) {
      const int b = i % kSBuf;
      const uint32_t tS = tbase + b * 128 + lane_off;
      FP_TMARK(7);
      mbar_wait(&sm.s_full[b], (i / kSBuf) & 1);
      tc_fence_after();
      FP_TMARK(0);
      float v[64];
      tmem_ld_16x256b_x16(tS, reinterpret_cast<uint32_t*>(v));
      tmem_wait_ld();
      FP_TMARK(1);
      float alpha[2], rs[2];
      if (i == nk - 1)  // the diagonal block is the last one of the sorted row
        softmax_tile<true>(v, R0, a, scale_log2, m_used, alpha, rs);
      else
        softmax_tile<false>(v, R0, a, scale_log2, m_used, alpha, rs);
      FP_TMARK(2);
      l[0] = l[0] * alpha[0] + rs[0];
      l[1] = l[1] * alpha[1] + rs[1];
      // every PV completion is consumed (here, normally long complete): O then
      // holds sum_{t<i} P_t V_t and may be rescaled
      if (i > 0) mbar_wait(&sm.pv_done[(i - 1) % kSBuf], ((i - 1) / kSBuf) & 1);
      if (i > 0 && __any_sync(0xffffffffu, alpha[0] != 1.f || alpha[1] != 1.f)) {
        // rescale this thread's rows of O
        tc_fence_after();
        float ov[64];
        tmem_ld_16x256b_x16(tO, reinterpret_cast<uint32_t*>(ov));
        tmem_wait_ld();
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          ov[4 * k] *= alpha[0];
          ov[4 * k + 1] *= alpha[0];
          ov[4 * k + 2] *= alpha[1];
          ov[4 * k + 3] *= alpha[1];
        }
        tmem_st_16x256b_x16(tO, reinterpret_cast<uint32_t*>(ov));
      }
      FP_TMARK(4);
      // P (bf16 pairs): packed column 4k + a holds keys 8k + 2a, 8k + 2a + 1
      uint32_t pk[32];
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        pk[2 * k] = pack_bf16x2(v[4 * k], v[4 * k + 1]);
        pk[2 * k + 1] = pack_bf16x2(v[4 * k + 2], v[4 * k + 3]);
      }
      tmem_st_16x128b_x16(tS, pk);
      tmem_wait_st();
      FP_TMARK(5);
      tc_fence_before();
      mbar_arrive(&sm.p_full[b]);
      FP_TMARK(6);
    }
#ifdef FP_TIMING
    if (timing_on) {
      for (int k = 0; k < 8; ++k) atomicAdd(&g_attn_timing[k], (unsigned long long)tacc[k]);
      atomicAdd(&g_attn_timing[8], (unsigned long long)nk);
    }
#endif
    // epilogue: O / l -> bf16 -> global
    const float il0 = 1.0f / quad_sum(l[0]), il1 = 1.0f / quad_sum(l[1]);
    mbar_wait(&sm.pv_done[(nk - 1) % kSBuf], ((nk - 1) / kSBuf) & 1);
    tc_fence_after();
    float ov[64];
    tmem_ld_16x256b_x16(tO, reinterpret_cast<uint32_t*>(ov));
    tmem_wait_ld();
    // rows past n (ragged last block, zero-filled Q) are not stored
    const int row0 = qb * 128 + R0;
    uint32_t* d0 = reinterpret_cast<uint32_t*>(o + toff(ol, h, row0)) + a;
    uint32_t* d1 = d0 + 4 * ol.rs;  // row R0 + 8 (rs elements = rs / 2 bf16 pairs per row)
    if (row0 < n) {
#pragma unroll
      for (int k = 0; k < 16; ++k) d0[4 * k] = pack_bf16x2(ov[4 * k] * il0, ov[4 * k + 1] * il0);
    }
    if (row0 + 8 < n) {
#pragma unroll
      for (int k = 0; k < 16; ++k) d1[4 * k] = pack_bf16x2(ov[4 * k + 2] * il1, ov[4 * k + 3] * il1);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 9) tmem_dealloc(tbase, 512);
}

}  // namespace

size_t attn_smem_bytes() { return sizeof(AttnSmem); }

cudaError_t launch_attn_v7(const Shape& s, const Layout& lay, const CUtensorMap& qmap,
                           const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                           const int32_t* row_ptr, const int32_t* col_idx, bool dense,
                           cudaStream_t st);

cudaError_t launch_attn_v8(const Shape& s, const Layout& lay, const CUtensorMap& qmap,
                           const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                           const int32_t* row_ptr, const int32_t* col_idx, bool dense,
                           const void* const* peer_o, int n_peer, cudaStream_t st);
cudaError_t launch_attn_b64(const Shape& s, const Layout& lay, const CUtensorMap& qmap,
                            const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                            const int32_t* row_ptr, const int32_t* col_idx, cudaStream_t st);
cudaError_t launch_attn_v9(const Shape& s, const Layout& lay, const CUtensorMap& qmap,
                           const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                           const int32_t* row_ptr, const int32_t* col_idx, bool dense,
                           cudaStream_t st);

// FP_ATTN_VERSION selects the kernel: 5 = this file (default), 7 = fp_attn7.cu
// (two warpgroups on interleaved 64-key streams; measured slower, see there),
// 8 = fp_attn8.cu (q-block pairs sharing K/V loads, ping-pong softmax),
// 9 = fp_attn9.cu (q-block pairs sharing K/V loads, v5's single-stream softmax)
#ifndef FP_ATTN_VERSION
#define FP_ATTN_VERSION 8
#endif
#define FP_ATTN_V5 (FP_ATTN_VERSION == 5)
int attn_kv_box_rows() { return FP_ATTN_VERSION == 7 ? 64 : 128; }

static cudaError_t launch_attn_v5(const Shape& s, const Layout& lay, const CUtensorMap& qmap,
                                  const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                                  const int32_t* row_ptr, const int32_t* col_idx, bool dense,
                                  cudaStream_t st);

cudaError_t launch_attn(const Shape& s, const WsLayout& L, void* ws, const Layout& lay,
                        const CUtensorMap& qmap, const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                        const int32_t* row_ptr, const int32_t* col_idx, bool dense,
                        const void* const* peer_o, int n_peer, cudaStream_t st) {
  (void)L;
  (void)ws;
  if (s.b != 128) {
    // dense causal attention does not depend on the block size: the 128 kernel
    if (dense) return launch_attn(make_shape(s.H, s.G, s.n, 128), L, ws, lay, qmap, kmap, vmap, o,
                                  row_ptr, col_idx, dense, peer_o, n_peer, st);
    if (n_peer > 0) return cudaErrorNotSupported;
    return launch_attn_b64(s, lay, qmap, kmap, vmap, o, row_ptr, col_idx, st);
  }
  if (FP_ATTN_VERSION == 8)
    return launch_attn_v8(s, lay, qmap, kmap, vmap, o, row_ptr, col_idx, dense, peer_o, n_peer, st);
  if (n_peer > 0) return cudaErrorNotSupported;  // the fused output exchange is v8's
  if (FP_ATTN_V5) return launch_attn_v5(s, lay, qmap, kmap, vmap, o, row_ptr, col_idx, dense, st);
  if (FP_ATTN_VERSION == 9)
    return launch_attn_v9(s, lay, qmap, kmap, vmap, o, row_ptr, col_idx, dense, st);
  return launch_attn_v7(s, lay, qmap, kmap, vmap, o, row_ptr, col_idx, dense, st);
}

static cudaError_t launch_attn_v5(const Shape& s, const Layout& lay, const CUtensorMap& qmap,
                                  const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                                  const int32_t* row_ptr, const int32_t* col_idx, bool dense,
                                  cudaStream_t st) {
  static bool attr_done = false;
  const size_t smem = attn_smem_bytes();
  if (!attr_done) {
    cudaFuncSetAttribute(attn_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(attn_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_done = true;
  }
  const float scale_log2 = (1.0f / sqrtf(128.0f)) * kLog2e;
  const dim3 grid(s.H * s.nb);
  if (dense)
    attn_kernel<true><<<grid, kAttnThreads, smem, st>>>(qmap, kmap, vmap,
                                                        reinterpret_cast<__nv_bfloat16*>(o), lay.o,
                                                        lay.q.per, lay.k.per, s.H, s.G, s.n, s.nb, s.tri, row_ptr, col_idx,
                                                        scale_log2);
  else
    attn_kernel<false><<<grid, kAttnThreads, smem, st>>>(qmap, kmap, vmap,
                                                         reinterpret_cast<__nv_bfloat16*>(o), lay.o,
                                                         lay.q.per, lay.k.per, s.H, s.G, s.n, s.nb, s.tri, row_ptr, col_idx,
                                                         scale_log2);
  return cudaGetLastError();
}

}  // namespace fp

#ifdef FP_TIMING
extern "C" int fp_debug_attn_timing(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_attn_timing, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_attn_timing, z, sizeof(z));
  }
  return 0;
}
#endif
