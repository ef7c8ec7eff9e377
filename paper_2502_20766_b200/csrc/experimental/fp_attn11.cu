// EXPERIMENT (round 1), NOT BUILT: a CTA-pair (cta_group::2, M = 256)
// attention kernel, kept as the starting point for the next round.
// Status, measured on B200 (profiles/r01_v11_experiment.txt):
//   * correct: matches the default kernel (v8) to bf16 rounding on C1 and C2
//     (dense and sparse; max |diff| 0.002-0.016) -- after two barrier-phase
//     fixes: p_full per S buffer (a CTA's warpgroups can run ahead of the
//     peer's) and pv_done per buffer (a waiter can lag a barrier by two PVs,
//     beyond what one parity bit resolves);
//   * slower: C3 38.5 vs 32.9 ms sparse, 122.8 vs 113.3 ms dense. Three S
//     buffers hide the MMA latency (S wait 207-350 cycles per entry), but the
//     two warpgroups exponentiate the two halves of the SAME tile at the same
//     time, so each SM spends 1,024 MUFU cycles + ~570 of ld/max/exchange/
//     pack/store per tile with nothing overlapping the non-MUFU part (v8's
//     ping-pong overlaps it); and at C3 the pair computes every union entry
//     for both rows (1.18x the MMAs). Next: exp2 partly on the FMA pipe (the
//     FMA pipe is idle here) and staggering the warpgroups.
// To try it: add it to build.py SOURCES, route launch_attn to
// launch_attn_v11 (FP_ATTN_VERSION 11) and build the K tensor map with 64-row
// boxes (K is loaded in 64-key halves).
// fp_attn11.cu -- stage (iii) of FlexPrefill, y = A(Q, K, V, S) (P:66-83,
// P:287-288), version 11: a CTA PAIR (cluster of 2, cta_group::2 MMAs) per
// q-block pair, one query row per SM, S triple-buffered, one O.
//
// Why (profiles/r01_v8_phase_timing.txt, r01_dense_vs_cudnn.txt): in v8 each
// of the two rows of a CTA has ONE S buffer in TMEM (S_A, S_B, O_A, O_B fill
// all 512 columns), so S(e+1) of a row waits for that row's softmax(e) and
// PV(e): the MMA pipeline alone (softmax disabled) runs at 3147 cycles per
// union entry against 2048 of tensor work, and v8 ends at ~1650 cycles per
// computed tile. Here the two rows sit on the two SMs of a cluster and every
// MMA is one M = 256 cta_group::2 instruction: each SM holds its own 128 query
// rows, HALF of each K tile (64 keys) and HALF of each V tile (64 of the 128
// head dims), so
//   * each SM's TMEM holds only its own row: S0, S1, S2 (three S buffers)
//     and O; S(e) is issued two entries ahead of its softmax;
//   * K/V bytes per SM per entry halve (16 + 16 KiB) and so do the
//     tensor-core shared-memory operand reads of B.
// The two softmax warpgroups split every tile by keys (WG w: keys 64w..)
// and exchange half-row maxima through shared memory each entry (one running
// max, one O; WG w rescales and stores O's d-columns 64w..). Every union entry
// is computed for BOTH rows (one M = 256 MMA): an entry the row did not
// select gets P = 0 (no exponentials), so at C3 ~18% of the MMAs are spent
// on unselected (row, entry) pairs (tools/pair_study.py: 1.69 computed tiles
// per union entry); dense has one such tile per pair (the diagonal of row A).
//
// Roles (384 threads per CTA; the leader is cluster rank 0):
//   warps 0-3  softmax WG0 (keys 0-63 of each tile)    one query row per thread
//   warps 4-7  softmax WG1 (keys 64-127 of each tile)  (TMEM lane = row)
//   warp 8     K producer (own half: keys 64r..64r+63 of the block)
//   warp 9     TMEM allocation (both CTAs); MMA issuer (leader only)
//   warp 10    V producer (own half: head dims 64r..64r+63)
// Barriers that gate the MMA (q/k/v full, p_full) live in the leader: both
// CTAs' TMA loads complete_tx there (cta_group::2 TMA form) and both CTAs'
// softmax warps arrive there (remote arrive). Barriers the MMA releases (k/v
// empty, s_full, pv_done) are in both CTAs: the commits multicast.
#include <math.h>

#include "fp_common.cuh"
#include "fp_internal.h"

#ifdef FP_TIMING
// clock64 phase accumulators (tools/attn8_timing.py --v11): [0..2] softmax
// thread 0 of each WG (leader CTA), [8..12] the MMA issuer, [14] entries
__device__ unsigned long long g_attn11_timing[16];
#define FP_T11(k) do { if (t_on) { long long _t = clock64(); tacc[k] += _t - tlast; tlast = _t; } } while (0)
#define FP_T11_DECL(on) const bool t_on = (on); long long tacc[16] = {0}; long long tlast = clock64()
#define FP_T11_FLUSH(lo, hi) do { if (t_on) for (int _k = lo; _k < hi; ++_k) atomicAdd(&g_attn11_timing[_k], (unsigned long long)tacc[_k]); } while (0)
#else
#define FP_T11(k) do { } while (0)
#define FP_T11_DECL(on) do { } while (0)
#define FP_T11_FLUSH(lo, hi) do { } while (0)
#endif

namespace fp {

namespace {

constexpr int kThreads11 = 384;
constexpr int kKS11 = 4, kVS11 = 4;          // K / V ring depths (half tiles)
constexpr int kHalfBytes = kTileBytes / 2;   // 16 KiB: 64 keys x 128 d, or 128 keys x 64 d
constexpr uint32_t kColS11 = 0, kColO11 = 384;  // S0 S1 S2 | O
constexpr float kRescale11 = 8.0f;

struct Attn11Smem {
  uint8_t q[kTileBytes];              // own 128 query rows (two 128x64 SW128 boxes)
  uint8_t k[kKS11][kHalfBytes];       // two 64x64 boxes (d 0-63, d 64-127)
  uint8_t v[kVS11][kHalfBytes];       // one 128x64 box (head dims 64r..64r+63)
  uint64_t q_full;
  uint64_t k_full[kKS11], k_empty[kKS11];
  uint64_t v_full[kVS11], v_empty[kVS11];
  // three S buffers (entry e in buffer e % 3): S(e) is issued two entries ahead
  uint64_t s_full[3], p_full[2][3], pv_done[3];
  // per-entry half-row maxima [e & 3][WG][row]: a WG can be up to three
  // entries ahead of the other (unselected entries have no barrier)
  float mxs[4][2][128];
  float lsum[2][128];                 // final partial sums [WG][row]
  uint32_t tmem_base;
};

FP_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
FP_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same smem variable in CTA `rank`
FP_DEV uint32_t map_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
FP_DEV void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
// TMA 4-D box into this CTA's smem; completion bytes counted on the LEADER's barrier
FP_DEV void tma2_load_4d(void* dst, const CUtensorMap* m, uint32_t bar_cluster, int c0, int c1, int c2,
                         int c3, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1, {%3, %4, %5, %6}], [%2], %7;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "l"(pol)
      : "memory");
}
// wait with cluster-scope acquire (arrivals come from the peer CTA's threads)
FP_DEV void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  const long long t0 = clock64();
  while (true) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.b32 %0, 1, 0, P1;\n\t}"
        : "=r"(ok)
        : "r"(addr), "r"(parity)
        : "memory");
    if (ok) return;
    if (clock64() - t0 > (1ll << 34)) __trap();
  }
}
FP_DEV void umma_commit_mc(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b16 m;\n\tmov.b16 m, 3;\n\t"
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], m;\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
FP_DEV void tmem_alloc2(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
}
FP_DEV void tmem_dealloc2(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
FP_DEV float fmax3_11(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
FP_DEV void ffma2_11(float& d0, float& d1, float a0, float a1, float b, float c) {
  asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %4};\n\tmov.b64 rc, {%5, %5};\n\t"
      "fma.rn.f32x2 rd, ra, rb, rc;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b), "f"(c));
}
FP_DEV void fadd2_11(float& d0, float& d1, float a0, float a1, float b0, float b1) {
  asm("{\n\t.reg .b64 ra, rb, rd;\n\t"
      "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\t"
      "add.rn.f32x2 rd, ra, rb;\n\tmov.b64 {%0, %1}, rd;\n\t}"
      : "=f"(d0), "=f"(d1)
      : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
FP_DEV void tmem_ld_x64_11(uint32_t taddr, uint32_t* r) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x64.b32 " FP_REGLIST64 ", [%64];" : FP_R64(r) : "r"(taddr));
}

// S = Q K^T for both rows of the pair: M = 256 (128 rows per CTA), N = 128
// keys (64 per CTA), 8 k-steps. A: Q, K-major SW128, 2 boxes of 16 KiB (k-step
// kk at box kk/4, +32 B per step); B: K half, K-major SW128, 2 boxes of 8 KiB.
FP_DEV void umma2_ss_chain8(uint32_t d, uint64_t a0, uint64_t b0, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %9, %17, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %2, %10, %17, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %3, %11, %17, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %4, %12, %17, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %5, %13, %17, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %6, %14, %17, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %7, %15, %17, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %8, %16, %17, p;\n\t}" ::"r"(d),
      "l"(a0), "l"(a0 + 2), "l"(a0 + 4), "l"(a0 + 6), "l"(a0 + 1024), "l"(a0 + 1026), "l"(a0 + 1028),
      "l"(a0 + 1030), "l"(b0), "l"(b0 + 2), "l"(b0 + 4), "l"(b0 + 6), "l"(b0 + 512), "l"(b0 + 514),
      "l"(b0 + 516), "l"(b0 + 518), "r"(idesc));
}
// O += P V for both rows: M = 256, N = 128 head dims (64 per CTA), 8 k-steps
// of 16 keys. A = P in TMEM (bf16 pairs over S), B = V half (MN-major SW128,
// one 128x64 box: k-step kk at +2048 B).
FP_DEV void umma2_ts_chain8(uint32_t d, uint32_t a0, uint64_t b0, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, 1, 0;\n\tsetp.ne.b32 q, %18, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %9, %17, q;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%2], %10, %17, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%3], %11, %17, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%4], %12, %17, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%5], %13, %17, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%6], %14, %17, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%7], %15, %17, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%8], %16, %17, p;\n\t}" ::"r"(d),
      "r"(a0), "r"(a0 + 8), "r"(a0 + 16), "r"(a0 + 24), "r"(a0 + 32), "r"(a0 + 40), "r"(a0 + 48),
      "r"(a0 + 56), "l"(b0), "l"(b0 + 128), "l"(b0 + 256), "l"(b0 + 384), "l"(b0 + 512),
      "l"(b0 + 640), "l"(b0 + 768), "l"(b0 + 896), "r"(idesc), "r"(acc0));
}

// Half of O += P V (64 keys, 4 k-steps) for both rows.
FP_DEV void umma2_ts_chain4(uint32_t d, uint32_t a0, uint64_t b0, uint32_t idesc, uint32_t acc0) {
  asm volatile(
      "{\n\t.reg .pred p, q;\n\tsetp.ne.b32 p, 1, 0;\n\tsetp.ne.b32 q, %10, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %5, %9, q;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%2], %6, %9, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%3], %7, %9, p;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%4], %8, %9, p;\n\t}" ::"r"(d),
      "r"(a0), "r"(a0 + 8), "r"(a0 + 16), "r"(a0 + 24), "l"(b0), "l"(b0 + 128), "l"(b0 + 256),
      "l"(b0 + 384), "r"(idesc), "r"(acc0));
}

// Merge of the two rows' sorted key-block lists (as v8): bit 0 row A, bit 1 row B.
struct UnionIter11 {
  const int32_t* la;
  const int32_t* lb;
  int na, nb_, ia, ib;
  bool dense;
  FP_DEV bool done() const { return ia >= na && ib >= nb_; }
  FP_DEV int next(int& mask) {
    const int ka = ia < na ? (dense ? ia : __ldg(la + ia)) : 0x7fffffff;
    const int kb = ib < nb_ ? (dense ? ib : __ldg(lb + ib)) : 0x7fffffff;
    const int k = min(ka, kb);
    mask = (ka == k ? 1 : 0) | (kb == k ? 2 : 0);
    ia += mask & 1;
    ib += mask >> 1;
    return k;
  }
};

template <bool DENSE>
__global__ void __launch_bounds__(kThreads11, 1)
    attn11_kernel(const __grid_constant__ CUtensorMap qmap, const __grid_constant__ CUtensorMap kmap,
                  const __grid_constant__ CUtensorMap vmap, __nv_bfloat16* __restrict__ o,
                  const TLayout ol, int Hp, int Gp, int H, int G, int n, int nb, long long cap,
                  const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col_idx,
                  float scale_log2) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  if (smem_u32(smem_raw) & 1023u) __trap();
  Attn11Smem& sm = *reinterpret_cast<Attn11Smem*>(smem_raw);

  const int tid = threadIdx.x;
  const int wid = warp_id();
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  // work item (as v8): KV-group-major, q-block pairs descending
  const int item = blockIdx.x >> 1;
  const int gsz = H / G;
  const int npair = (nb + 1) >> 1;
  const int per_group = gsz * npair;
  const int g = item / per_group;
  const int rem = item - g * per_group;
  const int qbA = nb - 1 - 2 * (rem / gsz);
  const int qbB = qbA - 1;  // -1: no row B (the CTA of rank 1 then only feeds zeros)
  const int h = g * gsz + rem % gsz;
  const int qbX = rank == 0 ? qbA : qbB;
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

  if (wid == 9) tmem_alloc2(&sm.tmem_base, 512);
  if (tid == 256) {
    tma_prefetch_desc(&qmap);
    tma_prefetch_desc(&kmap);
    tma_prefetch_desc(&vmap);
    mbar_init(&sm.q_full, 1);
    for (int s = 0; s < kKS11; ++s) {
      mbar_init(&sm.k_full[s], 1);
      mbar_init(&sm.k_empty[s], 1);
    }
    for (int s = 0; s < kVS11; ++s) {
      mbar_init(&sm.v_full[s], 1);
      mbar_init(&sm.v_empty[s], 1);
    }
    for (int i = 0; i < 3; ++i) {
      mbar_init(&sm.s_full[i], 1);
      mbar_init(&sm.pv_done[i], 1);
      // 4 softmax warps of WG w in each of the 2 CTAs; one barrier per S
      // buffer: a CTA's WGs may run up to two entries ahead of the peer's
      mbar_init(&sm.p_full[0][i], 8);
      mbar_init(&sm.p_full[1][i], 8);
    }
    mbar_fence_init();
  }
  tc_fence_before();
  cluster_sync_all();  // barriers of both CTAs initialised, TMEM allocated
  tc_fence_after();
  const uint32_t tbase = sm.tmem_base;

  if (wid >= 8) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 88;");
    if (wid == 8 || wid == 10) {
      // ------------------------------------------------ TMA producers (both CTAs)
      if (lane_id() == 0) {
        const bool isK = (wid == 8);
        const uint64_t pol = policy_evict_last();
        const HeadCoord kc = head_coord(g, Gp);
        if (isK) {
          const HeadCoord qc = head_coord(h, Hp);
          const uint32_t qbar = map_rank(&sm.q_full, 0);
          if (leader) mbar_arrive_expect_tx(&sm.q_full, 2 * kTileBytes);
          const int qrow = max(qbX, 0) * 128;  // rank 1 of an odd tail loads any valid rows
          tma2_load_4d(sm.q, &qmap, qbar, 0, qrow, qc.h, qc.b, pol);
          tma2_load_4d(sm.q + kBoxBytes, &qmap, qbar, 64, qrow, qc.h, qc.b, pol);
        }
        const int depth = isK ? kKS11 : kVS11;
        uint64_t* full = isK ? sm.k_full : sm.v_full;
        uint64_t* empty = isK ? sm.k_empty : sm.v_empty;
        UnionIter11 it{la, lb, nA, nB, 0, 0, DENSE};
        int e = 0;
        for (; !it.done(); ++e) {
          int mask;
          const int kb = it.next(mask);
          const int s = e % depth;
          if (e >= depth) mbar_wait(&empty[s], ((e - depth) / depth) & 1);
          const uint32_t fbar = map_rank(&full[s], 0);
          if (leader) mbar_arrive_expect_tx(&full[s], 2 * kHalfBytes);
          if (isK) {
            // keys [128 kb + 64 rank, +64), both head-dim boxes (64-row map)
            tma2_load_4d(sm.k[s], &kmap, fbar, 0, kb * 128 + 64 * (int)rank, kc.h, kc.b, pol);
            tma2_load_4d(sm.k[s] + kHalfBytes / 2, &kmap, fbar, 64, kb * 128 + 64 * (int)rank, kc.h, kc.b, pol);
          } else {
            // all 128 keys, head dims [64 rank, +64) (128-row map)
            tma2_load_4d(sm.v[s], &vmap, fbar, 64 * (int)rank, kb * 128, kc.h, kc.b, pol);
          }
        }
        // drain: every slot filled is released by a multicast commit; consume
        // those releases so no arrival targets this CTA after it exits
        for (int d = max(0, e - depth); d < e; ++d) mbar_wait(&empty[d % depth], (d / depth) & 1);
      }
    } else if (wid == 9 && leader) {
      // ------------------------------------------------ MMA issuer (leader CTA)
      if (lane_id() == 0) {
        constexpr uint32_t idesc_s = make_idesc_bf16(256, 128, false);
        constexpr uint32_t idesc_o = make_idesc_bf16(256, 128, true);
        const uint64_t qdesc = sdesc_kmajor(smem_u32(sm.q), 0);
        FP_T11_DECL(true);
        auto issue_pv = [&](int e) {  // O += P(e) V(e): 8 k-steps, P of both halves at buffer cols 0..63
          const int vs = e % kVS11;
          const int bf = e % 3;
          FP_T11(12);
          mbar_wait(&sm.v_full[vs], (e / kVS11) & 1);
          FP_T11(9);
          mbar_wait(&sm.p_full[0][bf], (e / 3) & 1);
          FP_T11(10);
          mbar_wait(&sm.p_full[1][bf], (e / 3) & 1);
          FP_T11(11);
          tc_fence_after();
          umma2_ts_chain8(tbase + kColO11, tbase + kColS11 + bf * 128,
                          make_sdesc(smem_u32(sm.v[vs]), kBoxBytes, 1024), idesc_o, e >= 1);
          umma_commit_mc(&sm.pv_done[bf]);
          umma_commit_mc(&sm.v_empty[vs]);
        };
        mbar_wait(&sm.q_full, 0);
        UnionIter11 it{la, lb, nA, nB, 0, 0, DENSE};
        int e = 0;
        for (; !it.done(); ++e) {
          int mask;
          it.next(mask);
          const int ks = e % kKS11;
          FP_T11(12);
          mbar_wait(&sm.k_full[ks], (e / kKS11) & 1);
          FP_T11(8);
#ifdef FP_TIMING
          ++tacc[14];
#endif
          tc_fence_after();
          // S(e) overwrites P(e - 3) in buffer e % 3: PV(e - 3) was issued in
          // the previous iteration (one in-order tcgen05.mma stream)
          umma2_ss_chain8(tbase + kColS11 + (e % 3) * 128, qdesc, make_sdesc(smem_u32(sm.k[ks]), 16, 1024),
                          idesc_s);
          umma_commit_mc(&sm.s_full[e % 3]);
          umma_commit_mc(&sm.k_empty[ks]);
          if (e >= 2) issue_pv(e - 2);
        }
        if (e >= 2) issue_pv(e - 2);
        if (e >= 1) issue_pv(e - 1);
        FP_T11(12);
        FP_T11_FLUSH(8, 15);
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");
    // ------------------------------------------------ softmax warpgroups
    // WG w owns keys 64w..64w+63 of every S tile; the row max is combined
    // across the two WGs each entry (one running max, one O)
    const int w = wid >> 2;
    const int r = (wid & 3) * 32 + lane_id();  // query row within the block = TMEM lane
    const uint32_t lane_off = (uint32_t)((wid & 3) * 32) << 16;
    const uint32_t tO = tbase + kColO11 + lane_off;
    uint32_t pbar[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) pbar[i] = map_rank(&sm.p_full[w][i], 0);
    float m_used = -INFINITY, l = 0.f;
    UnionIter11 it{la, lb, nA, nB, 0, 0, DENSE};
    FP_T11_DECL(leader && (wid & 3) == 0 && lane_id() == 0);
    int e = 0;
    for (; !it.done(); ++e) {
      int mask;
      const int kb = it.next(mask);
      const int bf = e % 3;
      const uint32_t tSb = tbase + kColS11 + bf * 128 + lane_off;  // this buffer, lane base
      mbar_wait(&sm.s_full[bf], (e / 3) & 1);
      FP_T11(0);
      tc_fence_after();
      const bool sel = (mask >> rank) & 1;  // same for every thread of the CTA
      if (sel) {
        float v[64];
        tmem_ld_x64_11(tSb + 64 * w, reinterpret_cast<uint32_t*>(v));
        tmem_wait_ld();
        if (kb == qbX) {  // the diagonal block: keys 64w + c <= r only
#pragma unroll
          for (int c = 0; c < 64; ++c)
            if (64 * w + c > r) v[c] = -INFINITY;
        }
        float mc[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) mc[q] = fmax3_11(v[16 * q], v[16 * q + 1], v[16 * q + 2]);
#pragma unroll
        for (int c = 3; c < 15; c += 2)
#pragma unroll
          for (int q = 0; q < 4; ++q) mc[q] = fmax3_11(mc[q], v[16 * q + c], v[16 * q + c + 1]);
#pragma unroll
        for (int q = 0; q < 4; ++q) mc[q] = fmaxf(mc[q], v[16 * q + 15]);
        const float hm = fmaxf(fmaxf(mc[0], mc[1]), fmaxf(mc[2], mc[3]));
        // combine with the other half (both WGs have loaded S after this
        // barrier, so WG1 may then store its P over WG0's half of S)
        sm.mxs[e & 3][w][r] = hm;
        asm volatile("bar.sync 1, 256;" ::: "memory");
        const float mx = fmaxf(hm, sm.mxs[e & 3][w ^ 1][r]) * scale_log2;
        float alpha = 1.f;
        if (mx > m_used + kRescale11) {
          alpha = exp2f(m_used - mx);  // 0 on the first selected tile
          m_used = mx;
        }
        const float nm = -m_used;
        // rescale this WG's half of O (d-columns 64w..) before P(e) is
        // released; PV(e - 1) may still be in flight: wait for it
        if (e > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
          mbar_wait(&sm.pv_done[(e - 1) % 3], ((e - 1) / 3) & 1);
          tc_fence_after();
#pragma unroll
          for (int q2 = 0; q2 < 2; ++q2) {
            uint32_t ov[32];
            tmem_ld32(tO + 64 * w + q2 * 32, ov);
            tmem_wait_ld();
#pragma unroll
            for (int c = 0; c < 32; ++c) ov[c] = __float_as_uint(__uint_as_float(ov[c]) * alpha);
            tmem_st32(tO + 64 * w + q2 * 32, ov);
          }
        }
        float s0 = 0.f, s1 = 0.f, s2 = 0.f, s3 = 0.f;
#pragma unroll
        for (int ch = 0; ch < 2; ++ch) {
          const int c0 = ch * 32;
#pragma unroll
          for (int c = c0; c < c0 + 32; c += 2) ffma2_11(v[c], v[c + 1], v[c], v[c + 1], scale_log2, nm);
#pragma unroll
          for (int c = c0; c < c0 + 32; ++c) v[c] = fast_exp2(v[c]);
#pragma unroll
          for (int c = c0; c < c0 + 32; c += 4) {
            fadd2_11(s0, s1, s0, s1, v[c], v[c + 1]);
            fadd2_11(s2, s3, s2, s3, v[c + 2], v[c + 3]);
          }
          uint32_t pk[16];
#pragma unroll
          for (int c = 0; c < 16; ++c) pk[c] = pack_bf16x2(v[c0 + 2 * c], v[c0 + 2 * c + 1]);
          // P of keys 64w + c0.. at buffer columns 32w + c0/2 (bf16 pairs)
          tmem_st16(tSb + 32 * w + ch * 16, pk);
        }
        l = l * alpha + ((s0 + s1) + (s2 + s3));
        FP_T11(1);
      } else {
        // entry of the other row only: P = 0 for this row (the M = 256 MMA
        // covers both rows). WG1 writes over WG0's S half: fine, nobody reads
        // S of an unselected entry.
        uint32_t z[32];
#pragma unroll
        for (int c = 0; c < 32; ++c) z[c] = 0u;
        tmem_st32(tSb + 32 * w, z);
      }
      tmem_wait_st();
      FP_T11(2);
      tc_fence_before();
      __syncwarp();
      if (lane_id() == 0) mbar_arrive_remote(pbar[bf]);
      FP_T11(3);
    }
    FP_T11_FLUSH(0, 8);
#ifdef FP_TIMING
    if (t_on) atomicAdd(&g_attn11_timing[15], (unsigned long long)e);
#endif
    // ---- epilogue: l = l0 + l1 (same running max); WG w stores d-columns 64w..
    sm.lsum[w][r] = l;
    asm volatile("bar.sync 1, 256;" ::: "memory");
    if (qbX >= 0) {
      // the last PV of each buffer residue (entries b, b + 3, ... < e)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const int cnt = (e - b + 2) / 3;
        if (cnt > 0) mbar_wait(&sm.pv_done[b], (cnt - 1) & 1);
      }
      tc_fence_after();
      const float il = 1.0f / (sm.lsum[0][r] + sm.lsum[1][r]);
      const int row = qbX * 128 + r;
      const size_t off = toff(ol, h, row);
      uint4* dst = reinterpret_cast<uint4*>(o + off);
#pragma unroll
      for (int cb = 0; cb < 64; cb += 32) {
        uint32_t a[32];
        tmem_ld32(tO + 64 * w + cb, a);
        tmem_wait_ld();
        if (row < n) {
#pragma unroll
          for (int c = 0; c < 32; c += 8) {
            uint32_t wv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q)
              wv[q] = pack_bf16x2(__uint_as_float(a[c + 2 * q]) * il, __uint_as_float(a[c + 2 * q + 1]) * il);
            dst[(64 * w + cb + c) / 8] = make_uint4(wv[0], wv[1], wv[2], wv[3]);
          }
        }
      }
    }
  }
  tc_fence_before();
  cluster_sync_all();  // no CTA leaves while its peer may still signal it / use its TMEM
  if (wid == 9) tmem_dealloc2(tbase, 512);
}

}  // namespace

size_t attn11_smem_bytes() { return sizeof(Attn11Smem); }

#ifdef FP_TIMING
extern "C" int fp_debug_attn11_timing(unsigned long long* out, int reset) {
  cudaMemcpyFromSymbol(out, g_attn11_timing, sizeof(unsigned long long) * 16);
  if (reset) {
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_attn11_timing, z, sizeof(z));
  }
  return 0;
}
#endif

cudaError_t launch_attn_v11(const Shape& s, const Layout& lay, const CUtensorMap& qmap,
                            const CUtensorMap& kmap, const CUtensorMap& vmap, void* o,
                            const int32_t* row_ptr, const int32_t* col_idx, bool dense,
                            cudaStream_t st) {
  static bool attr_done = false;
  const size_t smem = attn11_smem_bytes();
  if (!attr_done) {
    cudaFuncSetAttribute(attn11_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(attn11_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(attn11_kernel<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    cudaFuncSetAttribute(attn11_kernel<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 0);
    attr_done = true;
  }
  const float scale_log2 = (1.0f / sqrtf(128.0f)) * kLog2e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2 * s.H * ((s.nb + 1) / 2));
  cfg.blockDim = dim3(kThreads11);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  auto* op = reinterpret_cast<__nv_bfloat16*>(o);
  if (dense)
    return cudaLaunchKernelEx(&cfg, attn11_kernel<true>, qmap, kmap, vmap, op, lay.o, lay.q.per, lay.k.per,
                              s.H, s.G, s.n, s.nb, s.tri, row_ptr, col_idx, scale_log2);
  return cudaLaunchKernelEx(&cfg, attn11_kernel<false>, qmap, kmap, vmap, op, lay.o, lay.q.per, lay.k.per,
                            s.H, s.G, s.n, s.nb, s.tri, row_ptr, col_idx, scale_log2);
}

}  // namespace fp
