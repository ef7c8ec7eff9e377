// fp_attn7.cu -- stage (iii) of FlexPrefill, y = A(Q, K, V, S) (P:66-83,
// P:287-288), version 7: two softmax warpgroups on interleaved key streams.
//
// STATUS: an experiment, NOT the default kernel (build with
// -DFP_ATTN_VERSION=7 to select it). It passes every parity test but is
// slower than v5 (C3 gamma 0.95: 46.6 vs 31-32 ms standalone): the S = Q K^T
// products become M=128 x N=64 MMAs, which cost ~44 cycles each instead of 32
// (tools/ubench_mma.cu), and the issuing thread, which now handles 24 MMAs
// and 8 commits per 128-key block, is the bottleneck (tools/attn7_timing.py:
// ~1500 cycles per 64-key sub-tile in the issuer, softmax warps waiting on S
// and P.V ~60% of the time). Kept for the measurements it documents.
//
// Why: in v5 (fp_attn.cu) all 8 softmax warps work on the same key tile at
// the same time, so the MUFU (exp2, 16/clk/SM) idles while every warp loads S,
// rescales O or stores P (tools/attn_timing.py: 1236 of 1867 cycles per tile in
// the exp phase, MUFU ~60% busy). Here each 128-key block of the row's CSR
// list is split into two 64-key sub-tiles; warpgroup A (warps 0-3) owns the
// first half of every block, warpgroup B (warps 4-7) the second half. Each
// warpgroup runs its own online softmax (running max, row sum, O accumulator)
// over its key stream, so the two warps of a scheduler are out of phase and
// one's non-exp work hides under the other's exponentials. The two partial
// results are merged once per row at the end (the log-sum-exp merge of two
// disjoint key sets, exact up to rounding).
//
// One CTA per (head, query block) work item, 384 threads:
//   warp 8   K producer    Q tile (128 rows) once, then K sub-tiles (64 keys) of
//                          the row's key blocks into a kStages TMA ring
//   warp 10  V producer    V sub-tiles into their own ring
//   warp 9   MMA issuer    Q -> TMEM once (tcgen05.cp); S_j = Q K_j^T (M=128,
//                          N=64, A operand in TMEM) into S[j&1]; O[j&1] += P_j V_j
//                          (M=128, N=128, K=64, P in TMEM). S_{j+2} is issued as
//                          soon as warpgroup (j&1) has LOADED S_j (P lives in its
//                          own TMEM columns), so S is always one sub-tile ahead.
//   warps 0-7 softmax      one query row per thread (32x32b TMEM shape): the row
//                          max / sum are thread-local; lazy rescale (2^8) as v5
// TMEM (512 columns): S_A [0,64) S_B [64,128) P_A [128,160) P_B [160,192)
//                     Q [192,256) O_A [256,384) O_B [384,512).
// The diagonal block (last in a sorted row) is sub-tiles 2nk-2 (A, keys +0..63)
// and 2nk-1 (B, keys +64..127) with the causal mask j <= i.
#include <math.h>

#include "fp_common.cuh"
#include "fp_internal.h"

#ifdef FP_TIMING
__device__ unsigned long long g_attn7_timing[32];
#define T7_MARK(k) do { if (t7_on) { long long _t = clock64(); t7[k] += _t - t7_last; t7_last = _t; } } while (0)
#define T7_DECL(cond) const bool t7_on = (cond); long long t7[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long t7_last = clock64();
#define T7_FLUSH(base) do { if (t7_on) for (int _k = 0; _k < 8; ++_k) atomicAdd(&g_attn7_timing[(base) + _k], (unsigned long long)t7[_k]); } while (0)
#else
#define T7_MARK(k) do { } while (0)
#define T7_DECL(cond)
#define T7_FLUSH(base) do { } while (0)
#endif

namespace fp {

namespace {

constexpr int kThreads7 = 384;
constexpr int kSubKeys = 64;
constexpr int kSubBytes = kSubKeys * 128 * 2;  // 16 KiB: two 64x64 SW128 boxes
constexpr int kSubBox = kSubBytes / 2;         // 8 KiB
constexpr int kStages7 = 5;                    // K and V ring depth (sub-tiles)
constexpr uint32_t kColS7 = 0, kColP7 = 128, kColQ7 = 192, kColO7 = 256;
constexpr float kRescale7 = 8.0f;  // lazy rescale: tolerate P up to 2^8 (as v5)

struct Attn7Smem {
  uint8_t q[kTileBytes];  // 32 KiB, 1024-B aligned (first member)
  uint8_t k[kStages7][kSubBytes];
  uint8_t v[kStages7][kSubBytes];
  uint64_t q_full;
  uint64_t k_full[kStages7], k_empty[kStages7];
  uint64_t v_full[kStages7], v_empty[kStages7];
  uint64_t s_full[2], s_free[2], p_full[2], pv_done[2];
  float m_x[2][128], l_x[2][128];  // final merge exchange
  uint32_t tmem_base;
};

FP_DEV float fmax3_7(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
FP_DEV void ffma2_7(float& d0, float& d1, float a0, float a1, float b, float c) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %4};\n\tmov.b64 rc, {%5, %5};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b), "f"(c));
}
FP_DEV void fadd2_7(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
// 32 lanes x 32b, 64 consecutive columns (one row per thread)
FP_DEV void tmem_ld_32x32b_x64(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 " FP_REGLIST64 ", [%64];"
               : FP_R64(r)
               : "r"(taddr));
}
// S = Q K^T for one 64-key sub-tile: 8 k-steps in ONE asm statement (one
// elect/uniform-operand wrapper instead of eight); A = Q in TMEM columns
// a0 + 8 kk, B descriptors b0 + koff(kk) precomputed by the caller.
FP_DEV void umma_s8(uint32_t d, uint32_t a0, uint64_t b0, uint32_t idesc) {
  constexpr uint64_t o1 = 32 >> 4, o2 = 64 >> 4, o3 = 96 >> 4, o4 = kSubBox >> 4;
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %9, %17, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %10, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%3], %11, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%4], %12, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%5], %13, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%6], %14, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%7], %15, %17, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%8], %16, %17, p;\n\t}" ::"r"(d),
      "r"(a0), "r"(a0 + 8), "r"(a0 + 16), "r"(a0 + 24), "r"(a0 + 32), "r"(a0 + 40), "r"(a0 + 48),
      "r"(a0 + 56), "l"(b0), "l"(b0 + o1), "l"(b0 + o2), "l"(b0 + o3), "l"(b0 + o4),
      "l"(b0 + o4 + o1), "l"(b0 + o4 + o2), "l"(b0 + o4 + o3), "r"(idesc));
}
// O += P V for one sub-tile: 4 k-steps (16 keys each) in one asm statement;
// A = P in TMEM columns a0 + 8 kk, B = V descriptor b0 + kk * 2048 B.
FP_DEV void umma_pv4(uint32_t d, uint32_t a0, uint64_t b0, uint32_t idesc, uint32_t acc_first) {
  constexpr uint64_t o = 2048 >> 4;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, 1, 0;\n\tsetp.ne.b32 q, %10, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %5, %9, q;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %6, %9, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%3], %7, %9, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%4], %8, %9, p;\n\t}" ::"r"(d),
      "r"(a0), "r"(a0 + 8), "r"(a0 + 16), "r"(a0 + 24), "l"(b0), "l"(b0 + o), "l"(b0 + 2 * o),
      "l"(b0 + 3 * o), "r"(idesc), "r"(acc_first));
}

// K sub-tile as the K-major B operand of S = Q K^T: k-step kk (16 of d) at box
// kk/4 (8 KiB boxes of 64 keys x 64 d), byte (kk%4)*32; SBO = 8 rows x 128 B.
FP_DEV uint64_t sdesc_k7(uint32_t saddr, int kk) {
  return make_sdesc(saddr + (kk >> 2) * kSubBox + (kk & 3) * 32, 16, 1024);
}
// V sub-tile as the MN-major B operand of O += P V: k-step kk = keys
// [16kk, 16kk+16) at +2048 B; LBO = the second 64-wide d box (8 KiB).
FP_DEV uint64_t sdesc_v7(uint32_t saddr, int kk) { return make_sdesc(saddr + kk * 2048, kSubBox, 1024); }

// 64-row sub-tile of flattened head hh, rows [row, row + 64), two 64x64 boxes
FP_DEV void tma_sub_hint(void* dst, const CUtensorMap* m, uint64_t* bar, int row, int hh, int per,
                         uint64_t pol) {
  const HeadCoord c = head_coord(hh, per);
  tma_load_4d_hint(dst, m, bar, 0, row, c.h, c.b, pol);
  tma_load_4d_hint(static_cast<char*>(dst) + kSubBox, m, bar, 64, row, c.h, c.b, pol);
}

template <bool DENSE>
__global__ void __launch_bounds__(kThreads7, 1)
    attn7_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                 const __grid_constant__ CUtensorMap vmap, __nv_bfloat16* __restrict__ o,
                 const TLayout ol, int Hp, int Gp, int H, int G, int n, int nb, long long cap,
                 const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                 float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (smem_u32(smem_raw) & 1023u) __trap();  // SW128 tiles need 1024-B alignment
  Attn7Smem& sm = *reinterpret_cast<Attn7Smem*>(smem_raw);

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
  const int ns = 2 * nk;  // sub-tiles

  if (wid == 9) tmem_alloc(&sm.tmem_base, 512);
  if (tid == 256) {
    tma_prefetch_desc(&qmap);
    tma_prefetch_desc(&kmap);
    tma_prefetch_desc(&vmap);
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < kStages7; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&sm.s_full[b], 1);
      mbar_init(&sm.s_free[b], 4);   // one arrival per warp of the group
      mbar_init(&sm.p_full[b], 4);
      mbar_init(&sm.pv_done[b], 1);
    }
    mbar_fence_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm.tmem_base;

  if (wid >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 56;");
    if (wid == 8 || wid == 10) {
      // ------------------------------------------------ TMA producers
      if (lane_id() == 0) {
        const bool isK = (wid == 8);
        const uint64_t pol = policy_evict_last();
        if (isK) {
          mbar_arrive_expect_tx(&sm.q_full, kTileBytes);
          tma_tile(sm.q, &qmap, &sm.q_full, qb * 128, h, Hp);
        }
        uint64_t* full = isK ? sm.k_full : sm.v_full;
        uint64_t* empty = isK ? sm.k_empty : sm.v_empty;
        const CUtensorMap* map = isK ? &kmap : &vmap;
        for (int j = 0; j < ns; ++j) {
          const int s = j % kStages7;
          const int kb = DENSE ? (j >> 1) : __ldg(list + (j >> 1));
          if (j >= kStages7) mbar_wait(&empty[s], ((j - kStages7) / kStages7) & 1);
          mbar_arrive_expect_tx(&full[s], kSubBytes);
          tma_sub_hint(isK ? sm.k[s] : sm.v[s], map, &full[s], kb * 128 + (j & 1) * 64, g, Gp, pol);
        }
      }
    } else if (wid == 9) {
      // ------------------------------------------------ MMA issuer
      if (lane_id() == 0) {
        constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, false);
        constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, true);
        const uint32_t qa = smem_u32(sm.q);
        T7_DECL(blockIdx.x % 64 == 0)
        auto issue_s = [&](int j) {
          const int s = j % kStages7, b = j & 1;
          T7_MARK(4);
          mbar_wait(&sm.k_full[s], (j / kStages7) & 1);
          T7_MARK(0);
          // S[b] is free once the group has loaded S_{j-2} into registers
          if (j >= 2) mbar_wait(&sm.s_free[b], ((j - 2) >> 1) & 1);
          T7_MARK(1);
          tc_fence_after();
          umma_s8(tbase + kColS7 + b * 64, tbase + kColQ7, sdesc_k7(smem_u32(sm.k[s]), 0), idesc_s);
          umma_commit(&sm.s_full[b]);
          if (j + kStages7 < ns) umma_commit(&sm.k_empty[s]);
        };
        auto issue_pv = [&](int j) {
          const int s = j % kStages7, b = j & 1;
          T7_MARK(4);
          mbar_wait(&sm.v_full[s], (j / kStages7) & 1);
          T7_MARK(2);
          mbar_wait(&sm.p_full[b], (j >> 1) & 1);
          T7_MARK(3);
          tc_fence_after();
          umma_pv4(tbase + kColO7 + b * 128, tbase + kColP7 + b * 32, sdesc_v7(smem_u32(sm.v[s]), 0),
                   idesc_o, j >= 2);
          umma_commit(&sm.pv_done[b]);
          if (j + kStages7 < ns) umma_commit(&sm.v_empty[s]);
        };
        mbar_wait(&sm.q_full, 0);
        tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < 8; ++kk)  // Q (K-major SW128 in smem) -> TMEM columns kColQ7 + 8 kk
          asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tbase + kColQ7 + kk * 8),
                       "l"(sdesc_kmajor(qa, kk)));
        // order (matches the expected event order of two out-of-phase groups):
        // S0 S1 S2 | S3 PV0 | S4 PV1 | S5 PV2 | ...
        issue_s(0);
        issue_s(1);
        if (2 < ns) issue_s(2);
        for (int j = 0; j < ns; ++j) {
          if (j + 3 < ns) issue_s(j + 3);
          issue_pv(j);
        }
        T7_MARK(4);
#ifdef FP_TIMING
        if (t7_on) { t7[5] = ns; }
#endif
        T7_FLUSH(16);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 200;");
    // ------------------------------------------------ softmax warpgroups
    const int grp = wid >> 2;                   // 0 = A (first halves), 1 = B
    const int r = (wid & 3) * 32 + lane_id();   // query row within the block = TMEM lane
    const uint32_t lane_off = (uint32_t)((wid & 3) * 32) << 16;
    const uint32_t tS = tbase + kColS7 + grp * 64 + lane_off;
    const uint32_t tP = tbase + kColP7 + grp * 32 + lane_off;
    const uint32_t tO = tbase + kColO7 + grp * 128 + lane_off;
    const int c_off = grp * 64;  // key offset of this group's half inside a block
    float m_used = -INFINITY, l = 0.f;
    T7_DECL(blockIdx.x % 64 == 0 && (tid == 0 || tid == 128))
    for (int j = grp; j < ns; j += 2) {
      const int t = j >> 1;  // this group's sub-tile count so far
      T7_MARK(7);
      mbar_wait(&sm.s_full[grp], t & 1);
      T7_MARK(0);
      tc_fence_after();
      float v[64];
      tmem_ld_32x32b_x64(tS, reinterpret_cast<uint32_t*>(v));
      tmem_wait_ld();
      if (j + 2 < ns) {  // S[grp] may be overwritten by S_{j+2}
        tc_fence_before();
        __syncwarp();
        if (lane_id() == 0) mbar_arrive(&sm.s_free[grp]);
      }
      T7_MARK(1);
      const bool diag = (j >= ns - 2);
      if (diag) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (c_off + c > r) v[c] = -INFINITY;
      }
      float m0 = fmax3_7(v[0], v[1], v[2]), m1 = fmax3_7(v[3], v[4], v[5]);
#pragma unroll
      for (int c = 6; c < 62; c += 4) {
        m0 = fmax3_7(m0, v[c], v[c + 1]);
        m1 = fmax3_7(m1, v[c + 2], v[c + 3]);
      }
      const float mx = fmax3_7(m0, m1, fmaxf(v[62], v[63])) * scale_log2;
      float alpha = 1.f;
      if (mx > m_used + kRescale7) {
        alpha = exp2f(m_used - mx);  // 0 on the group's first sub-tile
        m_used = mx;
      }
      // a row can see no key of this group's sub-tile (diagonal, rows < 64 in B)
      const float nm = (m_used == -INFINITY) ? 0.f : -m_used;
#pragma unroll
      for (int c = 0; c < 64; c += 2) ffma2_7(v[c], v[c + 1], v[c], v[c + 1], scale_log2, nm);
#pragma unroll
      for (int c = 0; c < 64; ++c) v[c] = fast_exp2(v[c]);
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
      for (int c = 0; c < 64; c += 4) {
        fadd2_7(s0, s1, s0, s1, v[c], v[c + 1]);
        fadd2_7(s2, s3, s2, s3, v[c + 2], v[c + 3]);
      }
      l = l * alpha + ((s0 + s1) + (s2 + s3));
      uint32_t pk[32];
#pragma unroll
      for (int c = 0; c < 32; ++c) pk[c] = pack_bf16x2(v[2 * c], v[2 * c + 1]);
      T7_MARK(2);
      // O[grp] holds sum_{earlier} P V and P[grp] is free once PV_{j-2} is done
      if (j >= 2) {
        mbar_wait(&sm.pv_done[grp], ((j - 2) >> 1) & 1);
        T7_MARK(3);
        if (__any_sync(0xffffffffu, alpha != 1.f)) {
          tc_fence_after();
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint32_t ov[32];
            tmem_ld32(tO + q4 * 32, ov);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) * alpha);
            tmem_st32(tO + q4 * 32, ov);
          }
        }
      }
      T7_MARK(4);
      tmem_st32(tP, pk);
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&sm.p_full[grp]);
      T7_MARK(5);
    }
#ifdef FP_TIMING
    if (t7_on) t7[6] = (ns + 1 - grp) / 2;
#endif
    T7_FLUSH(grp * 8);
    // ---- merge the two groups' partial results: this thread finishes columns
    // [64 grp, 64 grp + 64) of row r from O_A and O_B
    const int jl = ns - 2 + grp;  // this group's last sub-tile
    mbar_wait(&sm.pv_done[grp], (jl >> 1) & 1);
    sm.m_x[grp][r] = m_used;
    sm.l_x[grp][r] = l;
    tc_fence_before();
    asm volatile("bar.sync 1, 256;" ::: "memory");
    tc_fence_after();
    const float mA = sm.m_x[0][r], mB = sm.m_x[1][r];
    const float m = fmaxf(mA, mB);  // finite: key qb*128 is visible to every row in A
    const float sA = exp2f(mA - m);
    const float sB = (mB == -INFINITY) ? 0.f : exp2f(mB - m);
    const float il = 1.0f / (sm.l_x[0][r] * sA + sm.l_x[1][r] * sB);
    const float fA = sA * il, fB = sB * il;
    const uint32_t tOA = tbase + kColO7 + lane_off + grp * 64;
    const int row = qb * 128 + r;
    uint4* dst = reinterpret_cast<uint4*>(o + toff(ol, h, row) + grp * 64);
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 32) {
      uint32_t ua[32], ub[32];
      tmem_ld32(tOA + c0, ua);
      tmem_ld32(tOA + 128 + c0, ub);
      tmem_wait_ld();
      if (row < n) {
#pragma unroll
        for (int c = 0; c < 32; c += 8) {
          uint32_t w[4];
#pragma unroll
          for (int e = 0; e < 4; ++e)
            w[e] = pack_bf16x2(__uint_as_float(ua[c + 2 * e]) * fA + __uint_as_float(ub[c + 2 * e]) * fB,
                               __uint_as_float(ua[c + 2 * e + 1]) * fA +
                                   __uint_as_float(ub[c + 2 * e + 1]) * fB);
          dst[(c0 + c) / 8] = make_uint4(w[0], w[1], w[2], w[3]);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 9) tmem_dealloc(tbase, 512);
}

}  // namespace

size_t attn7_smem_bytes() { return sizeof(Attn7Smem); }

cudaError_t launch_attn_v7(const Shape& s, const Layout& lay, const CUtensorMap& qmap,
                           const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                           const int32_t* row_ptr, const int32_t* col_idx, bool dense,
                           cudaStream_t st) {
  static bool attr_done = false;
  const size_t smem = attn7_smem_bytes();
  if (!attr_done) {
    cudaFuncSetAttribute(attn7_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(attn7_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attr_done = true;
  }
  const float scale_log2 = (1.0f / sqrtf(128.0f)) * kLog2e;
  const dim3 grid(s.H * s.nb);
  auto* op = reinterpret_cast<__nv_bfloat16*>(o);
  if (dense)
    attn7_kernel<true><<<grid, kThreads7, smem, st>>>(qmap, kmap, vmap, op, lay.o, lay.q.per,
                                                      lay.k.per, s.H, s.G, s.n, s.nb, s.tri,
                                                      row_ptr, col_idx, scale_log2);
  else
    attn7_kernel<false><<<grid, kThreads7, smem, st>>>(qmap, kmap, vmap, op, lay.o, lay.q.per,
                                                       lay.k.per, s.H, s.G, s.n, s.nb, s.tri,
                                                       row_ptr, col_idx, scale_log2);
  return cudaGetLastError();
}

}  // namespace fp

#ifdef FP_TIMING
extern "C" int fp_debug_attn7_timing(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_attn7_timing, sizeof(unsigned long long) * 32);
  if (reset) {
    unsigned long long z[32] = {0};
    cudaMemcpyToSymbol(g_attn7_timing, z, sizeof(z));
  }
  return 0;
}
#endif
