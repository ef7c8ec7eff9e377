// fp_attn8.cu -- stage (iii) of FlexPrefill, y = A(Q, K, V, S) (P:66-83,
// P:287-288), version 8: two query blocks of one head per CTA sharing their
// K/V loads, with two ping-ponging softmax warpgroups.
//
// Why: v5 (fp_attn.cu) fetches 64 KiB of K/V from L2 for every computed
// (q-block, k-block) tile. At C3 that is ~290 GB per launch, ~5.4 KB/cycle
// chip-wide, close to the measured L2 (LTS) throughput cap (~6.3 KB/cycle,
// B300_MICROARCH.md); ncu: 1820 cycles per tile per SM against 1024 of tensor
// work. Adjacent query blocks of a head select mostly the same key blocks
// (shared vertical columns; slash diagonals shifted by one), so a CTA that
// runs rows qb and qb-1 together loads each key block of the UNION of their
// lists once: tools/pair_study.py measured 0.58-0.60 union entries per
// computed tile on C3/C4/C5 (vs 1.0 in v5). The two rows' softmaxes are
// independent, so two warpgroups work on them out of phase (one
// exponentiates while the other loads S / stores P / rescales), the
// FlashAttention-4 ping-pong.
//
// One CTA per (head, q-block pair (qbA, qbB = qbA - 1)) work item, 384 threads:
//   warp 8   K producer   Q_A, Q_B tiles, then the K tiles of the union list
//                         (merge of the two sorted CSR rows) into a 3-stage ring
//   warp 10  V producer   the V tiles of the union list into a 2-stage ring
//   warp 9   MMA issuer   per union entry e and stream X in (A, B): first the
//                         pending O_X += P_X V (X's previous entry), then, if X
//                         selected e, S_X = Q_X K_e^T (both operands in smem,
//                         "SS"). Issue order per shared entry: PV_A S_A PV_B S_B,
//                         so the tensor core works for one stream while the
//                         other's softmax runs. A pending PV is issued no later
//                         than the next union entry (keeps the V ring moving:
//                         no deadlock when one row skips a run of entries).
//   warps 0-3 softmax A   one query row per thread (TMEM lane = row, 32x32b
//   warps 4-7 softmax B   shape, row max/sum thread-local); lazy running max as
//                         v5 (O rescaled in TMEM only when the max grows by
//                         > 2^8); P (bf16) over S; final O / l -> global.
// TMEM (512 columns): S/P_A [0,128) S/P_B [128,256) O_A [256,384) O_B [384,512).
// S_X of the next entry overwrites P_X right after PV_X is issued: one
// thread's tcgen05.mma stream executes in order (as in v5).
// Each row's diagonal block is the last of its own list and takes the
// intra-block causal mask. When nb is odd the last pair has no row B.
#include <math.h>

#include <algorithm>
#include <type_traits>

#include "fp_common.cuh"
#include "fp_internal.h"

#ifdef FP_TIMING
// clock64 phase accumulators (tools/attn8_timing.py): [0..5] softmax thread 0
// of each row, [8..12] the MMA issuer, [14] issuer entries, [15] softmax tiles
__device__ unsigned long long g_attn8_timing[20];
// [16] p_full arrival (thread 0 of the row) -> the issuer's wait returns,
// [17] S commit issued -> the row's softmax wait returns, [18] count of [16], [19] count of [17]
__device__ long long g_attn8_ts[148 * 4];
#define FP_T8(k) do { if (t_on) { long long _t = clock64(); tacc[k] += _t - tlast; tlast = _t; } } while (0)
#define FP_T8_DECL(on) const bool t_on = (on); long long tacc[20] = {0}; long long tlast = clock64()
#define FP_T8_FLUSH(lo, hi) do { if (t_on) for (int _k = lo; _k < hi; ++_k) atomicAdd(&g_attn8_timing[_k], (unsigned long long)tacc[_k]); } while (0)
#else
#define FP_T8(k) do { } while (0)
#define FP_T8_DECL(on) do { } while (0)
#define FP_T8_FLUSH(lo, hi) do { } while (0)
#endif

namespace fp {

namespace {

constexpr int kThreads8 = 384;
// K / V ring depths (tiles). A V slot is released by the entry's last PV,
// which the issuer sends no later than the next union entry, so two V slots
// cannot deadlock; the third K slot gives the K loads a second entry of lead
// (3 / 2 measured bitwise equal and 0.2-2% faster than 2 / 3 at C3, C4, C5
// 16k and dense: profiles/r02s3_attn_kv_ring_ab.txt)
#ifndef FP_KS8
#define FP_KS8 3
#endif
#ifndef FP_VS8
#define FP_VS8 2
#endif
constexpr int kKS8 = FP_KS8, kVS8 = FP_VS8;
// per-lane registers after setmaxnreg: producer / issuer warpgroup (dec) and
// the two softmax warpgroups (inc); the launch holds 12 warps x 168, so
// 4 x DEC + 8 x INC must stay <= 2016 (88 / 208, or 104 / 200)
#ifndef FP_DECREG8
#define FP_DECREG8 88
#endif
#ifndef FP_INCREG8
#define FP_INCREG8 208
#endif
static_assert(4 * FP_DECREG8 + 8 * FP_INCREG8 <= 12 * 168, "setmaxnreg budget");
#define FP_STR8_(x) #x
#define FP_STR8(x) FP_STR8_(x)
#ifndef FP_PV3
#define FP_PV3 1
#endif
constexpr bool kPv3 = FP_PV3 != 0;  // PV in three steps: keys 0-63 (p_lo), 64-95 (p_mid), 96-127 (p_full)
constexpr uint32_t kColS8 = 0, kColO8 = 256;
constexpr float kRescale8 = 8.0f;  // lazy rescale: tolerate P up to 2^8 (as v5)
// a row sum above 2^64 (some P may exceed 2^64 against the row's reference)
// flags the work item for an exact (max-first) redo
constexpr float kGuard8 = 18446744073709551616.0f;
// FMA-pipe exp2 (FlashAttention-4's MUFU offload, 16 or 32 of each row's 128
// exponentials per tile) was measured slower on every v8 variant (C3 gamma
// 0.95: 32.2 -> 34.9 / 38.0 ms; dense 112.5 -> 122.5 / 130.3 ms,
// profiles/r02_attn_nomax.txt) and is not built.
// P handed to the tensor core in two halves (keys 0-63, 64-127): the softmax
// stores P in 32-key chunks as the exponentials finish (tcgen05.st overlaps
// the next chunk's MUFU work) and arrives on p_lo once the first half is
// stored (checked after chunk 2's exponentials, so the wait does not stall), so
// the issuer starts PV's first four k-steps while the second half is still
// being exponentiated. Bitwise equal to the unsplit path; measured (C3,
// alternating 12-launch blocks) 34.04-34.19 ms vs 34.20-34.79 ms sparse, equal
// dense (profiles/r01_v8_phase_timing.txt). The gain is small because a row's
// period is bound by its single S buffer (S(e+1) waits for softmax(e) and
// PV(e)): the MMA pipeline alone runs at 3147 cycles per union entry against
// 2048 of tensor work (the -DFP_XSM8 experiment), see DESIGN.md section 6.

struct Attn8Smem {
  uint8_t q[2][kTileBytes];  // Q_A, Q_B (1024-B aligned: first member)
  uint8_t k[kKS8][kTileBytes];
  uint8_t v[kVS8][kTileBytes];
  uint64_t q_full, q_empty;
  uint64_t item_full[2], item_empty[2];  // work-item id ring (persistent scheduling)
  int item[2];
  uint64_t k_full[kKS8], k_empty[kKS8];
  uint64_t v_full[kVS8], v_empty[kVS8];
  uint64_t s_full[2], p_full[2], p_lo[2], p_mid[2], pv_done[2];
  uint32_t tmem_base;
  // exact redo of flagged work items (see the fetcher): ring written by the
  // softmax warps, read by the fetcher; per-item dedupe flags; completed
  // softmax-warp items (8 per item)
  int redo[8];
  int redo_tail, done_warps;
  unsigned redo_flag[8];
};
constexpr int kExact8 = 1 << 30;  // item id bit: recompute max-first on every tile

FP_DEV float fmax3_8(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
FP_DEV void ffma2_8(float& d0, float& d1, float a0, float a1, float b, float c) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %4};\n\tmov.b64 rc, {%5, %5};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b), "f"(c));
}
FP_DEV void fadd2_8(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
FP_DEV void tmem_ld_32x32b_x64_8(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 " FP_REGLIST64 ", [%64];"
               : FP_R64(r)
               : "r"(taddr));
}
FP_DEV void tmem_st_32x32b_x64_8(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x64.b32 [%64], " FP_REGLIST64 ";"
               :
               : FP_W64(r), "r"(taddr));
}

// The MMA issuer runs as a whole warp (FP_WARPISSUE8, default): every lane
// executes the same loop on the same (warp-uniform) values and the MMA /
// commit instructions are predicated on elect.sync inside the asm. With the
// issuer under `if (lane_id() == 0)` instead, the descriptors live in
// per-thread registers and ptxas wraps every tcgen05.mma in an R2UR +
// elect/branch loop: ~52 cycles to issue one MMA (tools/attn8_timing.py),
// which made the single issuing thread the bottleneck of the kernel.
#define FP_ELECT "elect.sync _|ep, 0xffffffff;\n\t"
FP_DEV void umma_ss_chain8_w(uint32_t d, uint64_t a0, uint64_t b0, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p, ep;\n\tsetp.ne.b32 p, 1, 0;\n\t" FP_ELECT
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
FP_DEV void umma_pv_chain4_w(uint32_t d, uint32_t a0, uint64_t b0, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, q, ep;\n\tsetp.ne.b32 p, 1, 0;\n\tsetp.ne.b32 q, %10, 0;\n\t" FP_ELECT
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %5, %9, q;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %6, %9, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%3], %7, %9, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%4], %8, %9, p;\n\t}" ::"r"(d),
      "r"(a0), "r"(a0 + 8), "r"(a0 + 16), "r"(a0 + 24), "l"(b0), "l"(b0 + 128), "l"(b0 + 256),
      "l"(b0 + 384), "r"(idesc), "r"(acc0));
}
// two PV k-steps (accumulating), K = 16 keys each
FP_DEV void umma_pv_chain2_w(uint32_t d, uint32_t a0, uint64_t b0, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p, ep;\n\tsetp.ne.b32 p, 1, 0;\n\t" FP_ELECT
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %3, %5, p;\n\t"
      "@ep tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %4, %5, p;\n\t}" ::"r"(d),
      "r"(a0), "r"(a0 + 8), "l"(b0), "l"(b0 + 128), "r"(idesc));
}
FP_DEV void umma_commit_w(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred ep;\n\t" FP_ELECT
      "@ep tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}

#define PVCHAIN4(...) umma_pv_chain4_w(__VA_ARGS__)
#define SSCHAIN8(...) umma_ss_chain8_w(__VA_ARGS__)
#define COMMIT8(b) umma_commit_w(b)

// Merge of the two rows' sorted key-block lists: next union entry.
// mask bit 0: row A selected it, bit 1: row B. The list heads are loaded one
// entry ahead, so the global-load latency overlaps the caller's work.
struct UnionIter {
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

// Block size 64 (reading A27): the attention runs on COARSE 128 x
// 128 tiles. Coarse row J holds the 64-row query blocks 2J and 2J+1 (one
// contiguous 128-row Q tile); its entries are the coarse key tiles m = kb / 2
// of the union of the two 64-rows' sorted lists, each with a 4-bit mask, bit
// 2 hx + hy = "query block 2J + hx selected key block 2m + hy". The softmax
// sets every unselected 64 x 64 quadrant of its rows to -inf, so exactly the
// selected blocks contribute; quadrants computed but masked are the price of
// the 128-wide tensor-core tile. The two 64-rows of a coarse row are adjacent
// in the 64-block CSR (row 2J+1 follows row 2J).
struct CoarseRow {
  const int32_t* l;  // row 2J's list; row 2J+1's follows it
  int n0, n1, i0, i1;
  FP_DEV void init(const int32_t* l_, int n0_, int n1_) {
    l = l_;
    n0 = n0_;
    n1 = n1_;
    i0 = i1 = 0;
  }
  FP_DEV bool done() const { return i0 >= n0 && i1 >= n1; }
  FP_DEV int peek() const {
    const int a = i0 < n0 ? (__ldg(l + i0) >> 1) : 0x7fffffff;
    const int b = i1 < n1 ? (__ldg(l + n0 + i1) >> 1) : 0x7fffffff;
    return min(a, b);
  }
  FP_DEV int next(int& mask) {  // coarse key tile m, quadrant mask
    const int m = peek();
    mask = 0;
    while (i0 < n0) {
      const int x = __ldg(l + i0);
      if ((x >> 1) != m) break;
      mask |= 1 << (x & 1);
      ++i0;
    }
    while (i1 < n1) {
      const int x = __ldg(l + n0 + i1);
      if ((x >> 1) != m) break;
      mask |= 4 << (x & 1);
      ++i1;
    }
    return m;
  }
};
// Union of the coarse rows A and B (mask bit 0: A has the tile, bit 1: B).
struct CoarseUnion {
  CoarseRow a, b;
  int ca, cb;
  FP_DEV void init(const int32_t* la, int na0, int na1, const int32_t* lb, int nb0, int nb1) {
    a.init(la, na0, na1);
    b.init(lb, nb0, nb1);
    ca = a.done() ? 0x7fffffff : a.peek();
    cb = b.done() ? 0x7fffffff : b.peek();
  }
  FP_DEV bool done() const { return ca == 0x7fffffff && cb == 0x7fffffff; }
  FP_DEV int next(int& mask) {
    const int k = min(ca, cb);
    mask = (ca == k ? 1 : 0) | (cb == k ? 2 : 0);
    int qm;
    if (mask & 1) {
      a.next(qm);
      ca = a.done() ? 0x7fffffff : a.peek();
    }
    if (mask & 2) {
      b.next(qm);
      cb = b.done() ? 0x7fffffff : b.peek();
    }
    return k;
  }
};

// One work item = (head h, q-block pair (qbA, qbB = qbA - 1)); items are
// numbered KV-group-major, pairs descending, heads of a group interleaved (the
// K/V of one group, 64 MiB at 128k, stay in L2 while its items run).
struct Item {
  int h, g, qbA, qbB, nA, nB;
  int nA1, nB1;  // COARSE: lengths of the second 64-rows (nA, nB: the first)
  const int32_t* la;
  const int32_t* lb;
};
template <bool DENSE, bool COARSE>
// order_gm = 0 (all K/V fit comfortably in L2, short n): pair-major over all
// heads, so every group's costliest pairs start in the first wave (a
// group-major order leaves the last groups' long rows as a tail).
FP_DEV Item decode_item(int item, int H, int G, int nb, long long cap, const int32_t* row_ptr,
                        const int32_t* col_idx, int order_gm, int nb64) {
  Item it;
  const int gsz = H / G;
  const int npair = (nb + 1) >> 1;
  if (order_gm) {
    const int per_group = gsz * npair;
    it.g = item / per_group;
    const int rem = item - it.g * per_group;
    it.qbA = nb - 1 - 2 * (rem / gsz);
    it.h = it.g * gsz + rem % gsz;
  } else {
    it.qbA = nb - 1 - 2 * (item / H);
    it.h = item % H;
    it.g = it.h / gsz;
  }
  it.qbB = it.qbA - 1;  // -1: no row B
  it.la = it.lb = nullptr;
  it.nA1 = it.nB1 = 0;
  if (COARSE) {
    // 64-block CSR (nb64 rows of 64 queries); coarse row J = 64-rows 2J, 2J+1
    const int32_t* rp = row_ptr + (size_t)it.h * (nb64 + 1);
    const int r0 = 2 * it.qbA;
    const int a0 = __ldg(rp + r0), a1 = __ldg(rp + r0 + 1);
    it.la = col_idx + (size_t)it.h * cap + a0;
    it.nA = a1 - a0;
    it.nA1 = r0 + 1 < nb64 ? __ldg(rp + r0 + 2) - a1 : 0;
    if (it.qbB >= 0) {
      const int b0 = __ldg(rp + r0 - 2), b1 = __ldg(rp + r0 - 1);
      it.lb = col_idx + (size_t)it.h * cap + b0;
      it.nB = b1 - b0;
      it.nB1 = a0 - b1;
    } else {
      it.nB = 0;
    }
  } else if (DENSE) {
    it.nA = it.qbA + 1;
    it.nB = it.qbB + 1;
  } else {
    const int32_t* rp = row_ptr + (size_t)it.h * (nb + 1);
    const int bA = __ldg(rp + it.qbA);
    it.nA = __ldg(rp + it.qbA + 1) - bA;
    it.la = col_idx + (size_t)it.h * cap + bA;
    if (it.qbB >= 0) {
      const int bB = __ldg(rp + it.qbB);
      it.nB = bA - bB;
      it.lb = col_idx + (size_t)it.h * cap + bB;
    } else {
      it.nB = 0;
    }
  }
  return it;
}

// Persistent: gridDim.x <= #SMs CTAs (one per SM), each runs work items until
// the list is exhausted. Items come from an atomic counter in the workspace
// (work_counter, zeroed before the launch: dynamic balancing, the next item
// goes to the first free SM). Without a workspace the grid has one CTA per
// item (item = blockIdx.x). Warp 8 fetches the ids and publishes them through a 2-slot
// ring (item_full / item_empty); every barrier phase below is counted
// cumulatively over the CTA's items. Across items: the next item's Q tiles
// are loaded once the last S MMA of the current one completed (q_empty), its
// first S MMAs run while the softmax warpgroups finish the current item, and
// a row's O is overwritten (first PV, accumulate = 0) only after its P -- which
// the warpgroup produces after its previous epilogue read O -- is stored.
// Softmax without a per-tile row-max pass (see the softmax warps): a row whose
// scores later exceed its reference by > 64 (log2) is flagged; its work item
// is pushed onto a CTA-local redo ring and the fetcher re-publishes it with
// kExact8 (every tile max-first) before taking new work, and before exiting
// waits until every published item has finished (done_warps) so late flags
// are still redone. The redo overwrites the item's output rows. sched
// (optional workspace scratch, zeroed before the launch): [0] work counter,
// [1] number of redone items (diagnostics).
template <bool DENSE, bool COARSE>
__global__ void __launch_bounds__(kThreads8, 1)
    attn8_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                 const __grid_constant__ CUtensorMap vmap, __nv_bfloat16* __restrict__ o,
                 const TLayout ol, int Hp, int Gp, int H, int G, int n, int nb, long long cap,
                 const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                 float scale_log2, const unsigned long long* __restrict__ peer_o, int n_peer,
                 int total_items, int* __restrict__ sched, int order_gm, int nb64) {
  FP_PDL_ENTRY();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (smem_u32(smem_raw) & 1023u) __trap();  // SW128 tiles need 1024-B alignment
  Attn8Smem& sm = *reinterpret_cast<Attn8Smem*>(smem_raw);

  const int tid = threadIdx.x;
  const int wid = warp_id();

  if (wid == 9) tmem_alloc(&sm.tmem_base, 512);
  if (tid == 256) {
    tma_prefetch_desc(&qmap);
    tma_prefetch_desc(&kmap);
    tma_prefetch_desc(&vmap);
    mbar_init(&sm.q_full, 1);
    mbar_init(&sm.q_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&sm.item_full[i], 1);
      mbar_init(&sm.item_empty[i], 10);  // V producer, issuer, 8 softmax warps
    }
    for (int s = 0; s < kKS8; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < kVS8; ++s) {
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 2);  // two commits per entry (see the issuer)
    }
    for (int x = 0; x < 2; ++x) {
      mbar_init(&sm.s_full[x], 1);
      mbar_init(&sm.p_full[x], 4);  // one arrival per softmax warp of the stream
      mbar_init(&sm.p_lo[x], 4);
      mbar_init(&sm.p_mid[x], 4);
      mbar_init(&sm.pv_done[x], 1);
    }
    mbar_fence_init();
    sm.redo_tail = sm.done_warps = 0;
    for (int i = 0; i < 8; ++i) sm.redo_flag[i] = 0, sm.redo[i] = -1;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tbase = sm.tmem_base;
  // consumers: the k-th item id of this CTA (-1: no more work). Lane 0 reads
  // the slot and broadcasts it, so the slot's only reader is the thread whose
  // item_empty arrival (release) orders the read before the producer's next
  // write of the slot.
  auto get_item = [&](int k) {
    int v = 0;
    if (lane_id() == 0) {
      mbar_wait(&sm.item_full[k & 1], (k >> 1) & 1);
      v = sm.item[k & 1];
    }
    return __shfl_sync(0xffffffffu, v, 0);
  };

  if (wid >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 " FP_STR8(FP_DECREG8) ";");
    if (wid == 8 || wid == 10) {
      // ------------------------------------------------ TMA producers (K: warp 8, V: warp 10)
      if (lane_id() == 0) {
        const bool isK = (wid == 8);
        const uint64_t pol = policy_evict_last();
        const int depth = isK ? kKS8 : kVS8;
        uint64_t* full = isK ? sm.k_full : sm.v_full;
        uint64_t* empty = isK ? sm.k_empty : sm.v_empty;
        const CUtensorMap* map = isK ? &kmap : &vmap;
        int e = 0;  // union entries loaded so far (all items)
        int redo_head = 0, n_new = 0;
        bool drained = false;
        for (int k = 0;; ++k) {
          int item;
          if (isK) {
            // scheduler: the k-th item of this CTA -- a flagged item to redo
            // first, else new work; when new work has run out, wait until all
            // published items finished (their flags are in) and exit when no
            // redo is pending
            volatile int* vtail = &sm.redo_tail;
            volatile int* vdone = &sm.done_warps;
            for (;;) {
              if (redo_head < *vtail) {
                // the pusher reserves its slot (tail) before writing it: wait
                // for the entry, then free the slot (-1); atomics on both sides
                int* slot = &sm.redo[redo_head++ & 7];
                while ((item = atomicOr(slot, 0)) < 0) __nanosleep(32);
                atomicExch(slot, -1);
                item |= kExact8;
                if (sched) atomicAdd(sched + 1, 1);
                break;
              }
              if (!drained) {
                item = sched ? atomicAdd(sched, 1) : (int)blockIdx.x + n_new * (int)gridDim.x;
                ++n_new;
                if (item < total_items) break;
                drained = true;
              }
              if (*vdone == 8 * k) {
                __threadfence_block();
                if (redo_head < *vtail) continue;
                item = -1;
                break;
              }
              __nanosleep(64);
            }
            if (k >= 2) mbar_wait(&sm.item_empty[k & 1], ((k - 2) >> 1) & 1);
            sm.redo_flag[k & 7] = 0;
            sm.item[k & 1] = item;
            mbar_arrive(&sm.item_full[k & 1]);
          } else {
            mbar_wait(&sm.item_full[k & 1], (k >> 1) & 1);  // V producer: lane 0 only
            item = sm.item[k & 1];
            mbar_arrive(&sm.item_empty[k & 1]);
          }
          if (item < 0) break;
          const Item it = decode_item<DENSE, COARSE>(item & ~kExact8, H, G, nb, cap, row_ptr, col_idx, order_gm, nb64);
          if (isK) {
            // Q_A, Q_B of this item once the previous item's S MMAs are done
            if (k >= 1) mbar_wait(&sm.q_empty, (k - 1) & 1);
            mbar_arrive_expect_tx(&sm.q_full, it.nB > 0 ? 2 * kTileBytes : kTileBytes);
            tma_tile(sm.q[0], &qmap, &sm.q_full, it.qbA * 128, it.h, Hp);
            if (it.nB > 0) tma_tile(sm.q[1], &qmap, &sm.q_full, it.qbB * 128, it.h, Hp);
          }
          typename std::conditional<COARSE, CoarseUnion, UnionIter>::type un;
          if constexpr (COARSE) un.init(it.la, it.nA, it.nA1, it.lb, it.nB, it.nB1);
          else un.init(it.la, it.lb, it.nA, it.nB, DENSE);
          for (; !un.done(); ++e) {
            int mask;
            const int kb = un.next(mask);
            const int s = e % depth;
            if (e >= depth) mbar_wait(&empty[s], ((e - depth) / depth) & 1);
            mbar_arrive_expect_tx(&full[s], kTileBytes);
            tma_tile_hint(isK ? sm.k[s] : sm.v[s], map, &full[s], kb * 128, it.g, Gp, pol);
          }
        }
        // drain: the issuer releases every slot it consumes (it does not know
        // the union length); consume those releases before the CTA exits
        for (int d = max(0, e - depth); d < e; ++d) mbar_wait(&empty[d % depth], (d / depth) & 1);
      }
    } else if (wid == 9) {
      // ------------------------------------------------ MMA issuer
      {  // the whole warp (elect.sync inside the MMA / commit asm)
        constexpr uint32_t idesc_s = make_idesc_bf16(128, 128, false);
        constexpr uint32_t idesc_o = make_idesc_bf16(128, 128, true);
        const uint64_t qdesc[2] = {sdesc_kmajor(smem_u32(sm.q[0]), 0), sdesc_kmajor(smem_u32(sm.q[1]), 0)};
        int cnt[2] = {0, 0};     // S tiles issued per stream (all items)
        int e = 0;               // union entries consumed (all items)
        FP_T8_DECL(lane_id() == 0);
        for (int k = 0;; ++k) {
          const int item = get_item(k);
          __syncwarp();
          if (lane_id() == 0) mbar_arrive(&sm.item_empty[k & 1]);
          if (item < 0) break;
          const Item itm = decode_item<DENSE, COARSE>(item & ~kExact8, H, G, nb, cap, row_ptr, col_idx, order_gm, nb64);
          int pend[2] = {-1, -1};  // union entry of X's S awaiting its PV
          int lcnt[2] = {0, 0};    // S tiles issued per stream in this item
          auto issue_pv = [&](int x) {
            const int ep = pend[x];
            const int vs = ep % kVS8;
            FP_T8(12);
            mbar_wait(&sm.v_full[vs], (ep / kVS8) & 1);
            FP_T8(9);
            const uint64_t vdesc = sdesc_mnmajor(smem_u32(sm.v[vs]), 0);
            mbar_wait(&sm.p_lo[x], (cnt[x] - 1) & 1);
            FP_T8(10);
            tc_fence_after();
            PVCHAIN4(tbase + kColO8 + x * 128, tbase + kColS8 + x * 128, vdesc, idesc_o, lcnt[x] > 1);
            FP_T8(12);
            if (kPv3) {  // k-steps 4-5 (keys 64-95) on p_mid
              mbar_wait(&sm.p_mid[x], (cnt[x] - 1) & 1);
              tc_fence_after();
              umma_pv_chain2_w(tbase + kColO8 + x * 128, tbase + kColS8 + x * 128 + 32, vdesc + 512, idesc_o);
            }
            mbar_wait(&sm.p_full[x], (cnt[x] - 1) & 1);
            FP_T8(11);
#ifdef FP_TIMING
            if (t_on) {
              tacc[16] += clock64() - *(volatile long long*)&g_attn8_ts[blockIdx.x * 4 + x];
            }
#endif
            tc_fence_after();
            if (kPv3) {
              umma_pv_chain2_w(tbase + kColO8 + x * 128, tbase + kColS8 + x * 128 + 48, vdesc + 768, idesc_o);
            } else {
              PVCHAIN4(tbase + kColO8 + x * 128, tbase + kColS8 + x * 128 + 32, vdesc + 512, idesc_o, 1);
            }
            COMMIT8(&sm.v_empty[vs]);
            COMMIT8(&sm.pv_done[x]);
            pend[x] = -1;
          };
          mbar_wait(&sm.q_full, k & 1);
          typename std::conditional<COARSE, CoarseUnion, UnionIter>::type un;
          if constexpr (COARSE) un.init(itm.la, itm.nA, itm.nA1, itm.lb, itm.nB, itm.nB1);
          else un.init(itm.la, itm.lb, itm.nA, itm.nB, DENSE);
          for (; !un.done(); ++e) {
            int mask;
            un.next(mask);
            const int ks = e % kKS8;
            FP_T8(12);
            mbar_wait(&sm.k_full[ks], (e / kKS8) & 1);
            FP_T8(8);
#ifdef FP_TIMING
            ++tacc[14];
#endif
            tc_fence_after();
            const uint64_t kdesc = sdesc_kmajor(smem_u32(sm.k[ks]), 0);
#pragma unroll
            for (int x = 0; x < 2; ++x) {
              if (pend[x] >= 0) issue_pv(x);
              if (mask & (1 << x)) {
                FP_T8(12);
                SSCHAIN8(tbase + kColS8 + x * 128, qdesc[x], kdesc, idesc_s);
                FP_T8(13);  // issue time of the 8 S MMAs
                COMMIT8(&sm.s_full[x]);
#ifdef FP_TIMING
                if (t_on) *(volatile long long*)&g_attn8_ts[blockIdx.x * 4 + 2 + x] = clock64();
#endif
                pend[x] = e;
                ++cnt[x];
                ++lcnt[x];
              }
            }
            COMMIT8(&sm.k_empty[ks]);
            // an entry only one row uses gets its second V-slot release here
            // (it arrives early, but the phase also needs the PV's commit)
            if (mask != 3) COMMIT8(&sm.v_empty[e % kVS8]);
          }
          // every S MMA of this item is issued: Q may be reloaded once they complete
          COMMIT8(&sm.q_empty);
          if (pend[0] >= 0) issue_pv(0);
          if (pend[1] >= 0) issue_pv(1);
        }
        FP_T8(12);
        FP_T8_FLUSH(8, 15);
        FP_T8_FLUSH(16, 17);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 " FP_STR8(FP_INCREG8) ";");
    // ------------------------------------------------ softmax warpgroups
    const int x = wid >> 2;                     // 0 = row A, 1 = row B
    const int r = (wid & 3) * 32 + lane_id();   // query row within the block = TMEM lane
    const uint32_t lane_off = (uint32_t)((wid & 3) * 32) << 16;
    const uint32_t tS = tbase + kColS8 + x * 128 + lane_off;
    const uint32_t tO = tbase + kColO8 + x * 128 + lane_off;
    int T = 0;  // tiles of this row processed in earlier items (barrier phases)
    FP_T8_DECL((wid & 3) == 0 && lane_id() == 0);
    for (int k = 0;; ++k) {
      const int item = get_item(k);
      __syncwarp();
      if (lane_id() == 0) mbar_arrive(&sm.item_empty[k & 1]);
      if (item < 0) break;
      const Item itm = decode_item<DENSE, COARSE>(item & ~kExact8, H, G, nb, cap, row_ptr, col_idx, order_gm, nb64);
      const bool exact = (item & kExact8) != 0;
      // COARSE: this row's own coarse entries (for the quadrant masks); the
      // tile count is only known when the walk ends
      CoarseRow crow;
      if (COARSE) crow.init(x ? itm.lb : itm.la, x ? itm.nB : itm.nA, x ? itm.nB1 : itm.nA1);
      const int nX = COARSE ? 0x7fffffff : (x ? itm.nB : itm.nA);
      const int qb = x ? itm.qbB : itm.qbA;
      float m_used = -INFINITY, l = 0.f;  // P = 2^(s * scale - m_used), l = sum of this thread's P
      int t = 0;
      for (; COARSE ? !crow.done() : t < nX; ++t) {
        int cmask = 15;
        const int cm = COARSE ? crow.next(cmask) : 0;
        const bool diag = COARSE ? cm == qb : t == nX - 1;
        const int ph = (T + t) & 1;  // this tile's phase of s_full / p_lo / p_full
        FP_T8(6);
        mbar_wait(&sm.s_full[x], ph);
        FP_T8(0);
#ifdef FP_TIMING
        if (t_on && t > 0) tacc[17] += clock64() - *(volatile long long*)&g_attn8_ts[blockIdx.x * 4 + 2 + x];
#endif
#ifdef FP_XSM8
        // experiment: softmax does no work (measures the MMA/issuer pipeline alone)
        tc_fence_after();
        __syncwarp();
        if (lane_id() == 0) { mbar_arrive(&sm.p_lo[x]); if (kPv3) mbar_arrive(&sm.p_mid[x]); mbar_arrive(&sm.p_full[x]); }
        continue;
#endif
        tc_fence_after();
        float v[128];
        tmem_ld_32x32b_x64_8(tS, reinterpret_cast<uint32_t*>(v));
        tmem_ld_32x32b_x64_8(tS + 64, reinterpret_cast<uint32_t*>(v + 64));
        // probe pv_done(t - 1) now (complete: S(t) followed PV(t - 1) in the
        // in-order MMA stream) so the probe's latency overlaps the TMEM load;
        // the phase is still consumed below, the loop only runs if it failed
        const bool pv_ok = t == 0 || mbar_try_wait(smem_u32(&sm.pv_done[x]), (T + t - 1) & 1);
        tmem_wait_ld();
        FP_T8(1);
        if (diag) {  // the diagonal block: keys j <= r only
#pragma unroll
          for (int c = 0; c < 128; ++c)
            if (c > r) v[c] = -INFINITY;
        }
        if (COARSE) {  // unselected 64 x 64 quadrants of this warp's 64-row half (warp-uniform)
          const int hx = r >> 6;
          if (!((cmask >> (2 * hx)) & 1)) {
#pragma unroll
            for (int c = 0; c < 64; ++c) v[c] = -INFINITY;
          }
          if (!((cmask >> (2 * hx + 1)) & 1)) {
#pragma unroll
            for (int c = 64; c < 128; ++c) v[c] = -INFINITY;
          }
        }
        if (!pv_ok) mbar_wait(&sm.pv_done[x], (T + t - 1) & 1);
        // Tiles after a row's first: no row-max pass (64 fmax3 per row and
        // tile plus the rescale vote; removing it measured -7% on C3, and every
        // variant that kept a per-tile check inside the exponential stream --
        // the max under the exponentials, guards on partial sums -- lost the
        // gain: profiles/r02_attn_nomax.txt). P = 2^(s * scale - m_used)
        // against the reference fixed by the row's first tile (exact softmax
        // up to rounding for any reference); the only hazard -- a later score
        // > 64 above it (log2), P near fp32 overflow -- is flagged per lane
        // once per row from the row sum (l <= 2^64 bounds every P; a larger,
        // infinite or NaN sum flags the row), and the whole work item is
        // redone max-first (kExact8) by this CTA. Max-first: a row's first
        // tile and every tile of a redone item; the reference moves to the
        // max if it grew by > 2^8.
        // COARSE: a thread whose first tiles were all masked has no reference
        // yet (m_used = -inf): its warp stays max-first until every lane has one
        const bool fast = t > 0 && !exact && (!COARSE || __all_sync(0xffffffffu, m_used > -INFINITY));
        float alpha = 1.f;
        if (!fast) {
          // row max of the raw scores: 8 independent fmax3 chains, then a tree
          constexpr int kJ = 16;
          float mc[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) mc[j] = fmax3_8(v[kJ * j], v[kJ * j + 1], v[kJ * j + 2]);
#pragma unroll
          for (int c = 3; c + 1 < kJ; c += 2)
#pragma unroll
            for (int j = 0; j < 8; ++j) mc[j] = fmax3_8(mc[j], v[kJ * j + c], v[kJ * j + c + 1]);
#pragma unroll
          for (int j = 0; j < 8; ++j) mc[j] = fmaxf(mc[j], v[kJ * j + kJ - 1]);
          const float mx =
              fmaxf(fmax3_8(mc[0], mc[1], mc[2]), fmax3_8(mc[3], mc[4], fmax3_8(mc[5], mc[6], mc[7]))) * scale_log2;
          if (mx > m_used + kRescale8) {
            alpha = exp2f(m_used - mx);  // 0 on the first tile
            m_used = mx;
          }
          if (t > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
            // O_X holds sum_{earlier} P V (PV(t - 1) is complete): rescale
            tc_fence_after();
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              uint32_t ov[32];
              tmem_ld32(tO + q * 32, ov);
              tmem_wait_ld();
#pragma unroll
              for (int c = 0; c < 32; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) * alpha);
              tmem_st32(tO + q * 32, ov);
            }
          }
        }
        // (a lane with no visible key so far: P = 2^-inf = 0)
        const float nm = COARSE && m_used == -INFINITY ? 0.f : -m_used;
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
          const int c0 = ch * 32;
#pragma unroll
          for (int c = c0; c < c0 + 32; c += 2) ffma2_8(v[c], v[c + 1], v[c], v[c + 1], scale_log2, nm);
#pragma unroll
          for (int c = c0; c < c0 + 32; ++c) v[c] = fast_exp2(v[c]);
#pragma unroll
          for (int c = c0; c < c0 + 32; c += 4) {
            fadd2_8(s0, s1, s0, s1, v[c], v[c + 1]);
            fadd2_8(s2, s3, s2, s3, v[c + 2], v[c + 3]);
          }
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) pk[c] = pack_bf16x2(v[c0 + 2 * c], v[c0 + 2 * c + 1]);
          if (ch == 2) {
            // p_lo after chunk 2's exponentials: the stores of chunks 0-1 have
            // completed by then, so the wait does not stall the MUFU stream
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane_id() == 0) mbar_arrive(&sm.p_lo[x]);
            FP_T8(4);
          }
          if (kPv3 && ch == 3) {
            // p_mid after chunk 3's exponentials: chunk 2 is stored, the
            // issuer runs PV k-steps 4-5 while chunk 3 is stored
            tmem_wait_st();
            tc_fence_before();
            __syncwarp();
            if (lane_id() == 0) mbar_arrive(&sm.p_mid[x]);
          }
          tmem_st16(tS + ch * 16, pk);  // P over S: 32 keys = 16 columns of bf16 pairs
        }
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
#ifdef FP_TIMING
        if (t_on) *(volatile long long*)&g_attn8_ts[blockIdx.x * 4 + x] = clock64();
#endif
        if (lane_id() == 0) mbar_arrive(&sm.p_full[x]);
        // the row sum after P is handed over (off the PV's critical path)
        l = fmaf(l, alpha, (s0 + s1) + (s2 + s3));
        FP_T8(5);
#ifdef FP_TIMING
        ++tacc[15];
#endif
      }
      const int ntl = t;  // tiles of this row in this item
      // overflow hazard of this row's P (checked on its row sum)
      const bool flag = __any_sync(0xffffffffu, !exact && ntl > 1 && !(l <= kGuard8));
      if (ntl > 0) {
        // epilogue: O / l -> bf16 -> global (rows past n are not stored)
        mbar_wait(&sm.pv_done[x], (T + ntl - 1) & 1);
        tc_fence_after();
        const float il = 1.0f / l;
        const int row = qb * 128 + r;
        const size_t off = toff(ol, itm.h, row);
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
        tc_fence_before();  // O reads complete before P of the next item is released
      }
      T += ntl;
      // a flagged item goes on the redo ring (once per item: the flag of its
      // slot dedupes the warps / rows that flag it), then the warp reports
      // the item done
      if (lane_id() == 0) {
        if (flag && atomicOr(&sm.redo_flag[k & 7], 1u) == 0) {
          atomicExch(&sm.redo[atomicAdd(&sm.redo_tail, 1) & 7], item & ~kExact8);
          __threadfence_block();  // the ring entry before the done count (rare: no fence otherwise)
        }
        atomicAdd(&sm.done_warps, 1);
      }
    }
    FP_T8_FLUSH(0, 8);
    FP_T8_FLUSH(17, 18);
#ifdef FP_TIMING
    if (t_on) atomicAdd(&g_attn8_timing[15], (unsigned long long)tacc[15]);
#endif
  }
  tc_fence_before();
  __syncthreads();
  if (wid == 9) tmem_dealloc(tbase, 512);
}

}  // namespace

size_t attn8_smem_bytes() { return sizeof(Attn8Smem); }

#ifdef FP_TIMING
extern "C" int fp_debug_attn8_timing(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_attn8_timing, sizeof(unsigned long long) * 20);
  if (reset) {
    unsigned long long z[20] = {0};
    cudaMemcpyToSymbol(g_attn8_timing, z, sizeof(z));
  }
  return 0;
}
#endif

// s: the 128-block shape (items = H * ceil(nb / 2) q-tile pairs). coarse: the
// CSR is a 64-block CSR of nb64 rows (capacity cap64 per head) walked as coarse
// 128 x 128 tiles with quadrant masks (block size 64, see CoarseRow).
cudaError_t launch_attn_v8(const Shape& s, const Layout& lay, const CUtensorMap& qmap,
                           const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                           const int32_t* row_ptr, const int32_t* col_idx, bool dense, bool coarse,
                           int nb64, long long cap64, const void* const* peer_o, int n_peer, int* sched,
                           cudaStream_t st) {
  const size_t smem = attn8_smem_bytes();
  cudaError_t ea = cudaSuccess;
  for (const void* f : {(const void*)attn8_kernel<true, false>, (const void*)attn8_kernel<false, false>,
                        (const void*)attn8_kernel<false, true>})
    if (ea == cudaSuccess) ea = ensure_smem_attr(f, smem);
  if (ea != cudaSuccess) return ea;
  int dev = 0, nsm = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const float scale_log2 = (1.0f / sqrtf(128.0f)) * kLog2e;
  const int total = s.H * ((s.nb + 1) / 2);
  // KV-group-major item order when the layer's K/V exceed half the L2 (one
  // group's K/V then stays resident while its items run), pair-major otherwise
  const int order_gm = (double)s.G * s.n * 128 * 2 * 2 > 64.0 * 1024 * 1024 ? 1 : 0;
  // persistent (one CTA per SM, dynamic work fetch) when a workspace holds the
  // scheduler; otherwise one CTA per item (a static round-robin over a
  // persistent grid would leave the per-item cost variance unbalanced)
  const dim3 grid(sched ? std::min(total, nsm) : total);
  if (sched) {
    const cudaError_t em = cudaMemsetAsync(sched, 0, 2 * sizeof(int), st);
    if (em != cudaSuccess) return em;
  }
  auto* op = reinterpret_cast<__nv_bfloat16*>(o);
  const auto* po = reinterpret_cast<const unsigned long long*>(peer_o);
  const long long cap = coarse ? cap64 : s.tri;
  const int nbr = coarse ? nb64 : s.nb;
  if (dense)
    FP_LAUNCH((attn8_kernel<true, false>), grid, kThreads8, smem, st, qmap, kmap, vmap, op, lay.o, lay.q.per,
              lay.k.per, s.H, s.G, s.n, s.nb, cap, row_ptr, col_idx, scale_log2, po, n_peer, total, sched,
              order_gm, nbr);
  else if (coarse)
    FP_LAUNCH((attn8_kernel<false, true>), grid, kThreads8, smem, st, qmap, kmap, vmap, op, lay.o, lay.q.per,
              lay.k.per, s.H, s.G, s.n, s.nb, cap, row_ptr, col_idx, scale_log2, po, n_peer, total, sched,
              order_gm, nbr);
  else
    FP_LAUNCH((attn8_kernel<false, false>), grid, kThreads8, smem, st, qmap, kmap, vmap, op, lay.o, lay.q.per,
              lay.k.per, s.H, s.G, s.n, s.nb, cap, row_ptr, col_idx, scale_log2, po, n_peer, total, sched,
              order_gm, nbr);
  return cudaGetLastError();
}

}  // namespace fp
