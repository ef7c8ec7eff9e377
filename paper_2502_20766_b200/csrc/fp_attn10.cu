// fp_attn10.cu -- stage (iii) of FlexPrefill, y = A(Q, K, V, S) (P:66-83,
// P:287-288), version 10: q-block pairs sharing their K/V loads (as v8,
// fp_attn8.cu), with the scores of each row double-buffered at half-tile
// granularity so a softmax warpgroup never waits for its next S.
//
// Why: in v8 each row has ONE S buffer of 128 TMEM columns (S_A, S_B, O_A,
// O_B fill the 512 columns), and P is written over S. S of the row's next
// key block can therefore only be issued after the softmax of the current
// one AND its P.V: per union entry a row spends ~2,100 cycles in the softmax
// plus ~1,100 waiting for PV + S on the tensor core, and the
// tensor pipe is ~58% busy. Here every 128-key block is processed as two
// 64-key halves and each row owns TWO 64-column S/P buffers plus its O:
//   TMEM: S_A0 [0,64) S_A1 [64,128) S_B0 [128,192) S_B1 [192,256)
//         O_A [256,384) O_B [384,512)
// The issuer keeps each row one half ahead: while the softmax works on half
// h (buffer h % 2), S of half h + 1 is already in the other buffer, and as
// soon as P(h) is stored the issuer runs PV(h) and then S(h + 2) into the
// buffer h just freed. A row's critical path is its softmax alone; the
// tensor core sees PV(h) + S(h + 2) of one row while the other row's softmax
// runs. The price is the N = 64 score MMA (~48 instead of 32 cycles per
// k-step: 384 + 256 cycles of tensor time per half and row instead of 512).
//
// One CTA per (head, q-block pair (qbA, qbB = qbA - 1)) work item, 384 threads:
//   warp 8   K producer   Q_A, Q_B tiles, then the K tiles of the union list
//   warp 10  V producer   the V tiles of the union list into a 3-stage ring
//   warp 9   MMA issuer   per union entry e and key half c, for each row X that
//                         selected e: PV of X's half two back (freeing its
//                         buffer), then S_X(e, c) = Q_X K_e[64c, 64c+64)^T
//   warps 0-3 softmax A   one query row per thread (TMEM lane = row, 32x32b
//   warps 4-7 softmax B   shape, row max / sum thread-local), lazy running
//                         max (O rescaled in TMEM only when the max grows by
//                         > 2^8), P (bf16) over S, final O / l -> global.
// The arithmetic per row is v8's with the keys of a block taken in two halves
// (the row max is the same; the row sum adds the halves' sums).
#include <math.h>

#include "fp_common.cuh"
#include "fp_internal.h"

#ifdef FP_TIMING
// clock64 phase accumulators (tools/attn10_timing.py): [0..4] softmax thread 0
// of each row, [8..13] the MMA issuer, [14] issuer entries, [15] softmax halves
__device__ unsigned long long g_attn10_timing[16];
#define FP_T10(k) do { if (t_on) { long long _t = clock64(); tacc[k] += _t - tlast; tlast = _t; } } while (0)
#define FP_T10_DECL(on) const bool t_on = (on); long long tacc[16] = {0}; long long tlast = clock64()
#define FP_T10_FLUSH(lo, hi) do { if (t_on) for (int _k = lo; _k < hi; ++_k) atomicAdd(&g_attn10_timing[_k], (unsigned long long)tacc[_k]); } while (0)
#define FP_T10_CNT(k) do { if (t_on) ++tacc[k]; } while (0)
#else
#define FP_T10(k) do { } while (0)
#define FP_T10_DECL(on) do { } while (0)
#define FP_T10_FLUSH(lo, hi) do { } while (0)
#define FP_T10_CNT(k) do { } while (0)
#endif

namespace fp {

namespace {

constexpr int kThreads10 = 384;
constexpr int kKS10 = 2, kVS10 = 3;  // K / V ring depths (tiles)
constexpr uint32_t kColS10 = 0, kColO10 = 256;
constexpr float kRescale10 = 8.0f;  // lazy rescale: tolerate P up to 2^8

struct Attn10Smem {
  uint8_t q[2][kTileBytes];  // Q_A, Q_B (1024-B aligned: first member)
  uint8_t k[kKS10][kTileBytes];
  uint8_t v[kVS10][kTileBytes];
  uint64_t q_full;
  uint64_t k_full[kKS10], k_empty[kKS10];
  uint64_t v_full[kVS10], v_empty[kVS10];
  uint64_t s_full[2][2], p_full[2][2], pv_done[2][2];  // [row][buffer]
  uint32_t tmem_base;
};

FP_DEV float fmax3_10(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
FP_DEV void ffma2_10(float& d0, float& d1, float a0, float a1, float b, float c) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %4};\n\tmov.b64 rc, {%5, %5};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b), "f"(c));
}
FP_DEV void fadd2_10(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
// 2^x for a pair on the FMA/ALU pipes (FlashAttention-4's MUFU offload):
// x = j + f (j = rint(x), |f| <= 1/2), 2^f by a degree-3 minimax polynomial
// (max rel. error 7.5e-5; P is rounded to bf16 afterwards, 2^-9), 2^j added
// into the exponent field. x is clamped at -125 (-inf -> 2^-125, and masked
// keys are zeroed separately).
FP_DEV void exp2_emu2_10(float x0, float x1, float& y0, float& y1) {
  const float kMagic = 12582912.0f;  // 1.5 * 2^23: rounds to an integer in the low mantissa bits
  x0 = fmaxf(x0, -125.0f);
  x1 = fmaxf(x1, -125.0f);
  float t0, t1, j0, j1, f0, f1, p0, p1;
  fadd2_10(t0, t1, x0, x1, kMagic, kMagic);
  fadd2_10(j0, j1, t0, t1, -kMagic, -kMagic);
  fadd2_10(f0, f1, x0, x1, -j0, -j1);
  ffma2_10(p0, p1, f0, f1, 0.0551716626f, 0.242611155f);
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %6};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(p0), "=f"(p1) : "f"(p0), "f"(p1), "f"(f0), "f"(f1), "f"(0.69326099f));
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %6};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(p0), "=f"(p1) : "f"(p0), "f"(p1), "f"(f0), "f"(f1), "f"(0.999928072f));
  y0 = __uint_as_float(__float_as_uint(t0) * 8388608u + __float_as_uint(p0));
  y1 = __uint_as_float(__float_as_uint(t1) * 8388608u + __float_as_uint(p1));
}
#ifndef FP_EMU10
#define FP_EMU10 0
#endif
constexpr int kEmu10 = FP_EMU10;  // exponentials per 32-key chunk on the FMA pipe

FP_DEV void tmem_ld_x64_10(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 " FP_REGLIST64 ", [%64];"
               : FP_R64(r)
               : "r"(taddr));
}

#define FP_ELECT10 "elect.sync _|ep, 0xffffffff;\n\t"
// S = Q K^T, M=128 N=64, 8 k-steps of 16 (operands K-major SW128, two 16 KiB
// boxes each: k-step kk at box kk/4, +32 B per step). Warp-wide, elect inside.
FP_DEV void umma_s64_chain8(uint32_t d, uint64_t a0, uint64_t b0, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p, ep;\n\tsetp.ne.b32 p, 1, 0;\n\t" FP_ELECT10
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %9, %17, 0;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %10, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], %3, %11, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], %4, %12, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], %5, %13, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], %6, %14, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], %7, %15, %17, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], %8, %16, %17, p;\n\t}" ::"r"(d),
      "l"(a0), "l"(a0 + 2), "l"(a0 + 4), "l"(a0 + 6), "l"(a0 + 1024), "l"(a0 + 1026),
      "l"(a0 + 1028), "l"(a0 + 1030), "l"(b0), "l"(b0 + 2), "l"(b0 + 4), "l"(b0 + 6),
      "l"(b0 + 1024), "l"(b0 + 1026), "l"(b0 + 1028), "l"(b0 + 1030), "r"(idesc));
}
// O += P V over 64 keys: 4 k-steps (16 keys each), A = P in TMEM columns
// a0 + 8 kk, B = V (MN-major SW128) descriptor b0 + kk * 2048 B.
FP_DEV void umma_pv64_chain4(uint32_t d, uint32_t a0, uint64_t b0, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, q, ep;\n\tsetp.ne.b32 p, 1, 0;\n\tsetp.ne.b32 q, %10, 0;\n\t" FP_ELECT10
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %5, %9, q;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %6, %9, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%3], %7, %9, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%4], %8, %9, p;\n\t}" ::"r"(d),
      "r"(a0), "r"(a0 + 8), "r"(a0 + 16), "r"(a0 + 24), "l"(b0), "l"(b0 + 128), "l"(b0 + 256),
      "l"(b0 + 384), "r"(idesc), "r"(acc0));
}
FP_DEV void umma_commit10(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred ep;\n\t" FP_ELECT10
      "@ep tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

// Merge of the two rows' sorted key-block lists: next union entry.
// mask bit 0: row A selected it, bit 1: row B. The list heads are loaded one
// entry ahead (the global-load latency overlaps the caller's work on the
// current entry instead of sitting on the issuer's critical path).
struct UnionIter10 {
  const int32_t* la;
  const int32_t* lb;
  int na, nb_, ia, ib;
  bool dense;
  int ca, cb;  // key blocks at ia / ib (INT_MAX past the end)
  FP_DEV void init(const int32_t* a_, const int32_t* b_, int na_, int nb2, bool d) {
    la = a_;
    lb = b_;
    na = na_;
    nb_ = nb2;
    ia = ib = 0;
    dense = d;
    ca = na > 0 ? (dense ? 0 : __ldg(la)) : 0x7fffffff;
    cb = nb_ > 0 ? (dense ? 0 : __ldg(lb)) : 0x7fffffff;
  }
  FP_DEV bool done() const { return ia >= na && ib >= nb_; }
  FP_DEV int next(int& mask) {
    const int k = min(ca, cb);
    mask = (ca == k ? 1 : 0) | (cb == k ? 2 : 0);
    if (mask & 1) {
      ++ia;
      ca = ia < na ? (dense ? ia : __ldg(la + ia)) : 0x7fffffff;
    }
    if (mask & 2) {
      ++ib;
      cb = ib < nb_ ? (dense ? ib : __ldg(lb + ib)) : 0x7fffffff;
    }
    return k;
  }
};

template <bool DENSE>
__global__ void __launch_bounds__(kThreads10, 1)
    attn10_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                  const __grid_constant__ CUtensorMap vmap, __nv_bfloat16* __restrict__ o,
                  const TLayout ol, int Hp, int Gp, int H, int G, int n, int nb, long long cap,
                  const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                  float scale_log2, const unsigned long long* __restrict__ peer_o, int n_peer) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (smem_u32(smem_raw) & 1023u) __trap();  // SW128 tiles need 1024-B alignment
  Attn10Smem& sm = *reinterpret_cast<Attn10Smem*>(smem_raw);

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
    for (int s = 0; s < kKS10; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 2);  // one release per row issuer
    }
    for (int s = 0; s < kVS10; ++s) {
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 4);  // two per row: its two PV halves, or two early releases
    }
    for (int x = 0; x < 2; ++x)
      for (int b = 0; b < 2; ++b) {
        mbar_init(&sm.s_full[x][b], 1);
        mbar_init(&sm.p_full[x][b], 4);  // one arrival per softmax warp of the row
        mbar_init(&sm.pv_done[x][b], 1);
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
        const int depth = isK ? kKS10 : kVS10;
        uint64_t* full = isK ? sm.k_full : sm.v_full;
        uint64_t* empty = isK ? sm.k_empty : sm.v_empty;
        const CUtensorMap* map = isK ? &kmap : &vmap;
        UnionIter10 it;
        it.init(la, lb, nA, nB, DENSE);
        int e = 0;
        for (; !it.done(); ++e) {
          int mask;
          const int kb = it.next(mask);
          const int s = e % depth;
          if (e >= depth) mbar_wait(&empty[s], ((e - depth) / depth) & 1);
          mbar_arrive_expect_tx(&full[s], kTileBytes);
          tma_tile_hint(isK ? sm.k[s] : sm.v[s], map, &full[s], kb * 128, g, Gp, pol);
        }
        // drain: every slot release is consumed before the CTA exits
        for (int d = max(0, e - depth); d < e; ++d) mbar_wait(&empty[d % depth], (d / depth) & 1);
      }
    } else {
      // ------------------------------------------------ MMA issuers: warp 9 row A, warp 11 row B
      // (whole warps, elect inside). Each issues only its own row's MMAs, so
      // one row's waits (its P, a V tile) never hold back the other row's
      // work; both streams share the tensor core.
      const int x = wid == 9 ? 0 : 1;
      constexpr uint32_t idesc_s = make_idesc_bf16(128, 64, false);
      constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, true);
      const uint64_t qdesc = sdesc_kmajor(smem_u32(sm.q[x]), 0);
      const uint32_t tSx = tbase + kColS10 + x * 128, tOx = tbase + kColO10 + x * 128;
      int sX = 0;   // halves whose S has been issued
      int pX = 0;   // halves whose PV has been issued
      int ent[2];   // [buffer] union entry of the half in that buffer
      FP_T10_DECL(lane_id() == 0);
      // PV of the oldest pending half (its P must be stored: p_full)
      auto issue_pv = [&]() {
        const int hh = pX, b = hh & 1, e = ent[b];
        const int vs = e % kVS10;
        FP_T10(13);
        mbar_wait(&sm.v_full[vs], (e / kVS10) & 1);
        FP_T10(9);
        mbar_wait(&sm.p_full[x][b], (hh >> 1) & 1);
        FP_T10(10);
        tc_fence_after();
        umma_pv64_chain4(tOx, tSx + b * 64, sdesc_mnmajor(smem_u32(sm.v[vs]), 0) + b * 512, idesc_o, hh > 0);
        umma_commit10(&sm.pv_done[x][b]);
        umma_commit10(&sm.v_empty[vs]);
        ++pX;
        FP_T10(12);
      };
      mbar_wait(&sm.q_full, 0);
      UnionIter10 it;
      it.init(la, lb, nA, nB, DENSE);
      for (int e = 0; !it.done(); ++e) {
        int mask;
        it.next(mask);
        const int ks = e % kKS10, vs = e % kVS10;
        if (mask & (1 << x)) {
          FP_T10(13);
          mbar_wait(&sm.k_full[ks], (e / kKS10) & 1);
          FP_T10(8);
          FP_T10_CNT(14);
          tc_fence_after();
          const uint64_t kdesc = sdesc_kmajor(smem_u32(sm.k[ks]), 0);
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const int b = sX & 1;
            // buffer b holds P of half sX - 2: its PV goes first (in-order stream)
            while (pX <= sX - 2) issue_pv();
            FP_T10(13);
            umma_s64_chain8(tSx + b * 64, qdesc, kdesc + c * 512, idesc_s);
            umma_commit10(&sm.s_full[x][b]);
            FP_T10(11);
            ent[b] = e;
            ++sX;
          }
          umma_commit10(&sm.k_empty[ks]);
        } else {
          // the row skips this entry: its pending PVs go now (the V ring keeps
          // moving), then its share of the slot releases -- after the slots
          // hold THIS entry (k_full / v_full), so an arrival never lands in a
          // slot's previous phase
          while (pX < sX) issue_pv();
          FP_T10(13);
          mbar_wait(&sm.k_full[ks], (e / kKS10) & 1);
          umma_commit10(&sm.k_empty[ks]);
          mbar_wait(&sm.v_full[vs], (e / kVS10) & 1);
          umma_commit10(&sm.v_empty[vs]);
          umma_commit10(&sm.v_empty[vs]);
          FP_T10(9);
        }
      }
      while (pX < sX) issue_pv();
      FP_T10(13);
      if (x == 0) FP_T10_FLUSH(8, 15);
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
    // ------------------------------------------------ softmax warpgroups
    const int x = wid >> 2;                     // 0 = row A, 1 = row B
    const int nX = x ? nB : nA;
    const int qb = x ? qbB : qbA;
    const int r = (wid & 3) * 32 + lane_id();   // query row within the block = TMEM lane
    const uint32_t lane_off = (uint32_t)((wid & 3) * 32) << 16;
    const uint32_t tS = tbase + kColS10 + x * 128 + lane_off;
    const uint32_t tO = tbase + kColO10 + x * 128 + lane_off;
    float m_used = -INFINITY, l = 0.f;
    const int nh = 2 * nX;
    FP_T10_DECL((wid & 3) == 0 && lane_id() == 0);
    float v[64];
    bool have = false;  // v already holds this half's S (prefetched)
    for (int hh = 0; hh < nh; ++hh) {
      const int b = hh & 1;
      const uint32_t tSb = tS + b * 64;
      FP_T10(4);
      if (!have) {
        mbar_wait(&sm.s_full[x][b], (hh >> 1) & 1);
        FP_T10(0);
        tc_fence_after();
        tmem_ld_x64_10(tSb, reinterpret_cast<uint32_t*>(v));
      }
      tmem_wait_ld();
      FP_T10_CNT(15);
      if (hh >= nh - 2) {  // the diagonal block (last entry): keys j <= r only
        const int c0 = (hh & 1) * 64;
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (c0 + c > r) v[c] = -INFINITY;
      }
      // row max of the half: 8 independent fmax3 chains, then a tree
      float mc[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) mc[j] = fmax3_10(v[8 * j], v[8 * j + 1], v[8 * j + 2]);
#pragma unroll
      for (int j = 0; j < 8; ++j) mc[j] = fmax3_10(mc[j], v[8 * j + 3], v[8 * j + 4]);
#pragma unroll
      for (int j = 0; j < 8; ++j) mc[j] = fmax3_10(mc[j], v[8 * j + 5], v[8 * j + 6]);
#pragma unroll
      for (int j = 0; j < 8; ++j) mc[j] = fmaxf(mc[j], v[8 * j + 7]);
      const float mx = fmaxf(fmax3_10(mc[0], mc[1], mc[2]), fmax3_10(mc[3], mc[4], fmax3_10(mc[5], mc[6], mc[7]))) *
                       scale_log2;
      float alpha = 1.f;
      if (mx > m_used + kRescale10) {
        alpha = exp2f(m_used - mx);  // 0 on the first half
        m_used = mx;
      }
      FP_T10(1);
      if (hh > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
        // O holds sum_{earlier halves} P V once PV(hh - 1) is done. (The
        // per-parity pv_done barriers cannot run two phases ahead of this
        // wait: PV(hh - 3) completed before S(hh - 1), PV(hh + 1) needs P of
        // half hh + 1, not produced yet -- so no phase needs consuming.)
        mbar_wait(&sm.pv_done[x][b ^ 1], ((hh - 1) >> 1) & 1);
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
      FP_T10(2);
      const float nm = -m_used;
      float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
      for (int ch = 0; ch < 2; ++ch) {
        const int c0 = ch * 32;
#pragma unroll
        for (int c = c0; c < c0 + 32; c += 2) ffma2_10(v[c], v[c + 1], v[c], v[c + 1], scale_log2, nm);
#pragma unroll
        for (int c = c0; c < c0 + 32 - kEmu10; ++c) v[c] = fast_exp2(v[c]);
#pragma unroll
        for (int c = c0 + 32 - kEmu10; c < c0 + 32; c += 2) exp2_emu2_10(v[c], v[c + 1], v[c], v[c + 1]);
        if (kEmu10 > 0 && hh >= nh - 2) {  // masked keys of the diagonal block: exactly 0
#pragma unroll
          for (int c = c0 + 32 - kEmu10; c < c0 + 32; ++c)
            if ((hh & 1) * 64 + c > r) v[c] = 0.f;
        }
#pragma unroll
        for (int c = c0; c < c0 + 32; c += 4) {
          fadd2_10(s0, s1, s0, s1, v[c], v[c + 1]);
          fadd2_10(s2, s3, s2, s3, v[c + 2], v[c + 3]);
        }
        uint32_t pk[16];
#pragma unroll
        for (int c = 0; c < 16; ++c) pk[c] = pack_bf16x2(v[c0 + 2 * c], v[c0 + 2 * c + 1]);
        tmem_st16(tSb + ch * 16, pk);  // P over S: 32 keys = 16 columns of bf16 pairs
      }
      l = l * alpha + ((s0 + s1) + (s2 + s3));
      // prefetch the next half's S if it is already complete (a non-blocking
      // probe: blocking here, before P(hh) is released, could deadlock when
      // the issuer needs PV(hh) to free a V slot first)
      have = false;
      if (hh + 1 < nh) {
        const bool rdy = mbar_try_wait(smem_u32(&sm.s_full[x][b ^ 1]), ((hh + 1) >> 1) & 1);
        if (__all_sync(0xffffffffu, rdy)) {
          tc_fence_after();
          tmem_ld_x64_10(tS + (b ^ 1) * 64, reinterpret_cast<uint32_t*>(v));
          have = true;
        }
      }
      tmem_wait_st();
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&sm.p_full[x][b]);
      FP_T10(3);
    }
    FP_T10(4);
    FP_T10_FLUSH(0, 5);
#ifdef FP_TIMING
    if (t_on) atomicAdd(&g_attn10_timing[15], (unsigned long long)tacc[15]);
#endif
    if (nX > 0) {
      // epilogue: O / l -> bf16 -> global (rows past n are not stored); the
      // last two PVs (one per buffer parity) are the ones still outstanding
      mbar_wait(&sm.pv_done[x][(nh - 2) & 1], ((nh - 2) >> 1) & 1);
      mbar_wait(&sm.pv_done[x][(nh - 1) & 1], ((nh - 1) >> 1) & 1);
      tc_fence_after();
      const float il = 1.0f / l;
      const int row = qb * 128 + r;
      const size_t off = toff(ol, h, row);
      uint4* dst = reinterpret_cast<uint4*>(o + off);
#pragma unroll
      for (int c0 = 0; c0 < 128; c0 += 32) {
        uint32_t ov[32];
        tmem_ld32(tO + c0, ov);
        tmem_wait_ld();
        if (row < n) {
          uint4 w4[4];
#pragma unroll
          for (int c = 0; c < 32; c += 8) {
            uint32_t w[4];
#pragma unroll
            for (int e = 0; e < 4; ++e)
              w[e] = pack_bf16x2(__uint_as_float(ov[c + 2 * e]) * il, __uint_as_float(ov[c + 2 * e + 1]) * il);
            w4[c / 8] = make_uint4(w[0], w[1], w[2], w[3]);
            dst[(c0 + c) / 8] = w4[c / 8];
          }
          // next row f4: the same row into every peer's output buffer (another
          // rank's buffer mapped into this process: the stores go over NVLink)
          for (int i = 0; i < n_peer; ++i) {
            uint4* pd = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(__ldg(peer_o + i)) + off);
#pragma unroll
            for (int c = 0; c < 4; ++c) pd[c0 / 8 + c] = w4[c];
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 9) tmem_dealloc(tbase, 512);
}

}  // namespace

#ifdef FP_TIMING
extern "C" int fp_debug_attn10_timing(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_attn10_timing, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_attn10_timing, z, sizeof(z));
  }
  return 0;
}
#endif

cudaError_t launch_attn_v10(const Shape& s, const Layout& lay, const CUtensorMap& qmap,
                            const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                            const int32_t* row_ptr, const int32_t* col_idx, bool dense,
                            const void* const* peer_o, int n_peer, cudaStream_t st) {
  const size_t smem = sizeof(Attn10Smem);
  cudaError_t ea = ensure_smem_attr((const void*)attn10_kernel<true>, smem);
  if (ea == cudaSuccess) ea = ensure_smem_attr((const void*)attn10_kernel<false>, smem);
  if (ea != cudaSuccess) return ea;
  const float scale_log2 = (1.0f / sqrtf(128.0f)) * kLog2e;
  const dim3 grid(s.H * ((s.nb + 1) / 2));
  auto* op = reinterpret_cast<__nv_bfloat16*>(o);
  if (dense)
    attn10_kernel<true><<<grid, kThreads10, smem, st>>>(qmap, kmap, vmap, op, lay.o, lay.q.per,
                                                        lay.k.per, s.H, s.G, s.n, s.nb, s.tri,
                                                        row_ptr, col_idx, scale_log2,
                                                        reinterpret_cast<const unsigned long long*>(peer_o),
                                                        n_peer);
  else
    attn10_kernel<false><<<grid, kThreads10, smem, st>>>(qmap, kmap, vmap, op, lay.o, lay.q.per,
                                                         lay.k.per, s.H, s.G, s.n, s.nb, s.tri,
                                                         row_ptr, col_idx, scale_log2,
                                                         reinterpret_cast<const unsigned long long*>(peer_o),
                                                         n_peer);
  return cudaGetLastError();
}

}  // namespace fp
