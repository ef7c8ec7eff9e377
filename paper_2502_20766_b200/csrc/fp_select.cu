// fp_select.cu -- stage (ii) of FlexPrefill: cumulative-attention index
// selection (Alg. 3; Alg. 4), forced first /
// diagonal key blocks and the minimum budget, emitted as a per-head
// block CSR for the attention kernel.
//
// Kernels:
//   topmass      N5  per segment (a_v, a_s of VS heads; flattened A_bar of QA
//                    heads): MSD radix *select by mass* on the fp32 bit
//                    patterns (11/11/10-bit digits) -> the threshold value
//                    lambda (Appendix B), ties -> lower index (A8),
//                    then an ordered compaction of the selected indices.
//                    Masses are summed in 2^-60 fixed point (uint64), so every
//                    sum is exact and order independent (deterministic).
//   topmass_rows f2  per query-block row of A_bar (qa_mode 1), row bitmaps
//   build_lines  N6a vertical-block / slash-diagonal bitmaps (A10 R1; R2 with vs_mode 1)
//   assemble     N6b per query-block row: rasterised lines or QA blocks,
//                    forced blocks (A11), minimum budget (A12)
//   row_scan     N6c per-head CSR row offsets + stats
//   write_cols   N6d CSR column indices (ascending kb)
#include <math.h>

#include <algorithm>

#include "fp_common.cuh"
#include "fp_internal.h"

namespace fp {

namespace {

constexpr int kSelThreads = 1024;
#ifdef FP_TM_TIMING
// globaltimer (ns) at phase boundaries of topmass_segment, thread 0 of each CTA:
// [head * 8 + cluster rank][phase] (tools/topmass_timing.py)
__device__ unsigned long long g_tm_t[512][16];
#define FP_TM(k) do { if (threadIdx.x == 0) { unsigned long long _t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(_t)); g_tm_t[blockIdx.y * 8 + blockIdx.x][k] = _t; } } while (0)
#else
#define FP_TM(k) do { } while (0)
#endif
constexpr float kFixScale = 1152921504606846976.0f;  // 2^60

// x (>= 0, finite) in 2^-60 fixed point, truncated: floor(min(x, 8) * 2^60),
// from the bit pattern (mantissa shifted by the exponent; no float->u64
// conversion unit): x = m * 2^(e - 150), m = 1.f (24 bits), so
// x * 2^60 = m << (e - 90) or m >> (90 - e).
__device__ __forceinline__ uint64_t fixp(float x) {
  const uint32_t b = __float_as_uint(fminf(x, 8.0f));
  const int e = (int)(b >> 23);
  if (e == 0) return 0;  // zero / denormals (< 2^-126): below 2^-60
  const uint64_t m = (uint64_t)((b & 0x7fffffu) | 0x800000u);
  const int sh = e - 90;
  return sh >= 0 ? (m << sh) : (sh > -64 ? (m >> -sh) : 0ull);
}

// block-wide inclusive scan of uint64 (1024 threads), returns inclusive value,
// *total gets the block total. Deterministic (integer).
__device__ uint64_t block_scan_u64(uint64_t v, uint64_t* wsum, uint64_t* total) {
  const int ln = lane_id(), w = warp_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t y = __shfl_up_sync(0xffffffffu, v, o);
    if (ln >= o) v += y;
  }
  if (ln == 31) wsum[w] = v;
  __syncthreads();
  if (w == 0) {
    uint64_t s = wsum[ln];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (ln >= o) s += y;
    }
    wsum[ln] = s;  // inclusive prefix of warp totals
  }
  __syncthreads();
  uint64_t add = (w > 0) ? wsum[w - 1] : 0;
  const uint64_t tot = wsum[31];
  __syncthreads();
  *total = tot;
  return v + add;
}

constexpr int kClMax = 8;  // max CTAs (one cluster) per head; chosen per launch
#ifndef FP_TOP_MIN_KEYS
#define FP_TOP_MIN_KEYS 16384
#endif
constexpr long long kTopMinKeys = FP_TOP_MIN_KEYS;  // scores per CTA below which more CTAs do not pay

// distributed shared memory helpers (thread block cluster)
__device__ __forceinline__ uint32_t cl_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cl_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t cl_map(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// remote loads are ordered by the cluster barriers around them (compiler
// barriers too), so they need no volatile / memory clobber: the compiler may
// issue a batch of them back to back (DSMEM latency ~200 cycles each)
__device__ __forceinline__ uint32_t cl_ld32(uint32_t a) {
  uint32_t v;
  asm("ld.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ unsigned long long cl_ld64(uint32_t a) {
  unsigned long long v;
  asm("ld.shared::cluster.u64 %0, [%1];" : "=l"(v) : "r"(a));
  return v;
}

struct TopSmem {
  uint32_t cnt[2048];             // this CTA's histogram of its slice
  unsigned long long mass[2048];
  uint32_t gcnt[2048];            // sub-group histogram (sum over the segment's CTAs)
  unsigned long long gmass[2048];
  uint64_t wsum[32];
  uint32_t found_bin;
  unsigned long long above_mass, above_cnt;
  unsigned long long slice_gt, slice_eq;  // compaction counts of this CTA's slice
};

// topmass(x[0..L), gamma) (A6-A8, Appendix B) by the nr CTAs of cluster ranks
// [r0, r0 + nr) (this CTA is rank r0 + sub); CTA `sub` owns the index slice
// [sub*S, (sub+1)*S), S = ceil(L / nr). Every CTA of the CLUSTER calls this the
// same number of times (it executes a fixed number of cluster barriers).
// MSD radix select by mass on the fp32 bit patterns (11/11/10-bit digits):
// per pass a count + fixed-point mass histogram of the keys that match the
// prefix found so far, merged over the sub-group through DSMEM, then the
// descending-digit scan finds the digit holding the threshold. Masses are
// sums of 2^-60 fixed-point values (exact, order independent).
__device__ void topmass_segment(TopSmem& sm, const float* __restrict__ x, long long L, int32_t* __restrict__ out,
                                float gamma, uint32_t r0, uint32_t nr, uint32_t sub, int32_t* count_out,
                                unsigned long long* mass_out) {
  const int tid = threadIdx.x;
  const long long S = (L + nr - 1) / nr;
  const long long lo = min(L, (long long)sub * S), hi = min(L, lo + S);
  unsigned long long T = 0, G = 0, rem = 0;
  bool count_mode = false;
  uint32_t prefix = 0, pmask = 0;
  unsigned long long above_mass_tot = 0, above_cnt_tot = 0;
  unsigned long long slice_gt = 0, slice_eq = 0;
  const int shifts[3] = {21, 10, 0};
  const int widths[3] = {11, 11, 10};
  FP_TM(0);
  for (int pass = 0; pass < 3; ++pass) {
    const int sh = shifts[pass];
    const uint32_t dmask = (1u << widths[pass]) - 1u;
    const int nbins = 1 << widths[pass];
    for (int b = tid; b < nbins; b += kSelThreads) {
      sm.cnt[b] = 0;
      sm.mass[b] = 0;
    }
    __syncthreads();
    FP_TM(1 + 4 * pass);
    // local histogram of the slice: 16-B loads of the 16-B-aligned body (4 in
    // flight per thread = 16 keys), the <= 3 keys before / after it scalar
    // shared atomics per digit run (integer: order independent): the count
    // an atomic add, the 64-bit fixed-point mass two native 32-bit adds on the
    // halves of mass[digit] (little endian) with the carry of the low one (a
    // 64-bit shared atomicAdd compiles to a CAS loop). Aggregating same-digit
    // lanes of a warp first (match + partial-mask reductions, a loop over the
    // warp's distinct digits) measured slower.
    auto flush = [&](uint32_t digit, uint32_t c, uint64_t f) {
      uint32_t* mh = reinterpret_cast<uint32_t*>(&sm.mass[digit]);
      atomicAdd(&sm.cnt[digit], c);
      const uint32_t lo = (uint32_t)f;
      const uint32_t old = atomicAdd(mh, lo);
      const uint32_t hi = (uint32_t)(f >> 32) + (old + lo < old ? 1u : 0u);
      if (hi) atomicAdd(mh + 1, hi);
    };
    auto hist_key = [&](uint32_t key) {
      if (key != 0xffffffffu && (key & pmask) == prefix) flush((key >> sh) & dmask, 1u, fixp(__uint_as_float(key)));
    };
    // eight adjacent keys of one thread: runs of equal digits are merged in
    // registers first (neighbouring scores share a digit often: fewer
    // same-address atomics, which the shared-memory unit serialises)
    auto hist_keys = [&](const uint4& k, const uint4& k2) {
      const uint32_t kk[8] = {k.x, k.y, k.z, k.w, k2.x, k2.y, k2.z, k2.w};
      uint32_t cd = 0xffffffffu, cc = 0;
      uint64_t cm = 0;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t key = kk[e];
        if (key == 0xffffffffu || (key & pmask) != prefix) continue;
        const uint32_t d = (key >> sh) & dmask;
        const uint64_t f = fixp(__uint_as_float(key));
        if (d == cd) {
          ++cc;
          cm += f;
        } else {
          if (cc) flush(cd, cc, cm);
          cd = d;
          cc = 1;
          cm = f;
        }
      }
      if (cc) flush(cd, cc, cm);
    };
    {
      const long long xmis = (long long)((reinterpret_cast<uintptr_t>(x) >> 2) & 3);
      const long long a0 = min(hi, lo + ((-(xmis + lo)) & 3));  // first 16-B-aligned key
      const long long nv = (hi - a0) / 4;                       // float4s of the body
      const long long a1 = a0 + 4 * nv;
      if (tid < a0 - lo) hist_key(__float_as_uint(__ldg(x + lo + tid)));
      if (tid < hi - a1) hist_key(__float_as_uint(__ldg(x + a1 + tid)));
      const float4* x4 = reinterpret_cast<const float4*>(x + a0);
      for (long long vb = 0; vb < nv; vb += 4 * kSelThreads) {
        // thread t: float4s 2t, 2t + 1 and 2048 + 2t, 2048 + 2t + 1 of the
        // step (eight adjacent keys per run merge)
        uint4 k4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const long long i = vb + (u >> 1) * 2 * kSelThreads + 2 * tid + (u & 1);
          if (i < nv) {
            const float4 f4 = __ldg(x4 + i);
            k4[u] = make_uint4(__float_as_uint(f4.x), __float_as_uint(f4.y), __float_as_uint(f4.z),
                               __float_as_uint(f4.w));
          } else {
            k4[u] = make_uint4(0xffffffffu, 0xffffffffu, 0xffffffffu, 0xffffffffu);
          }
        }
        hist_keys(k4[0], k4[1]);
        hist_keys(k4[2], k4[3]);
      }
    }
    FP_TM(2 + 4 * pass);
    if (nr > 1) {
      cl_sync();  // every CTA's local histogram is complete
      for (int b = tid; b < nbins; b += kSelThreads) {
        uint32_t cv[kClMax];
        unsigned long long mv[kClMax];
#pragma unroll
        for (uint32_t r = 0; r < kClMax; ++r) {
          if (r < nr) {
            cv[r] = cl_ld32(cl_map(&sm.cnt[b], r0 + r));
            mv[r] = cl_ld64(cl_map(&sm.mass[b], r0 + r));
          }
        }
        uint32_t c = 0;
        unsigned long long m = 0;
#pragma unroll
        for (uint32_t r = 0; r < kClMax; ++r)
          if (r < nr) {  // fixed order; integer sums are exact anyway
            c += cv[r];
            m += mv[r];
          }
        sm.gcnt[b] = c;
        sm.gmass[b] = m;
      }
      cl_sync();  // remote reads done before anyone clears its histogram
    } else {
      __syncthreads();
      for (int b = tid; b < nbins; b += kSelThreads) {
        sm.gcnt[b] = sm.cnt[b];
        sm.gmass[b] = sm.mass[b];
      }
      __syncthreads();
    }
    FP_TM(3 + 4 * pass);
    if (pass == 0) {
      // total mass T from the first-digit histogram (exact, fixed point)
      unsigned long long tl = 0;
      for (int b = tid; b < nbins; b += kSelThreads) tl += sm.gmass[b];
      uint64_t tot;
      block_scan_u64(tl, sm.wsum, &tot);
      T = tot;
      // K = min{k : C_k >= gamma T}  (A6, A7); G == 0 -> K = 1 (count mode)
      G = (unsigned long long)ceil((double)gamma * (double)T);
      count_mode = (G == 0);
      rem = count_mode ? 1ull : G;
      if (gamma >= 1.0f) {  // A7: gamma >= 1 selects everything (the passes still run,
        rem = 0;            // so every CTA of the cluster meets the same barriers)
      }
    }
    // descending-digit scan: thread t owns digits nbins-1-2t and nbins-2-2t
    const int d0 = nbins - 1 - 2 * tid, d1 = d0 - 1;
    uint64_t m0 = 0, m1 = 0, k0 = 0, k1 = 0;
    if (d0 >= 0) {
      m0 = sm.gmass[d0];
      k0 = sm.gcnt[d0];
    }
    if (d1 >= 0) {
      m1 = sm.gmass[d1];
      k1 = sm.gcnt[d1];
    }
    uint64_t tot;
    const uint64_t key_m = count_mode ? (k0 + k1) : (m0 + m1);
    const uint64_t other = count_mode ? (m0 + m1) : (k0 + k1);
    // both exclusive prefixes in one scan: key in the high, other in the low
    // 32 bits are not enough (masses are 64-bit), so two scans
    const uint64_t excl = block_scan_u64(key_m, sm.wsum, &tot) - key_m;
    const uint64_t excl_o = block_scan_u64(other, sm.wsum, &tot) - other;
    {
      const uint64_t q0 = count_mode ? k0 : m0, q1 = count_mode ? k1 : m1;
      const uint64_t o0 = count_mode ? m0 : k0;
      if (d0 >= 0 && excl < rem && rem <= excl + q0) {
        sm.found_bin = d0;
        sm.above_mass = count_mode ? excl_o : excl;
        sm.above_cnt = count_mode ? excl : excl_o;
      } else if (d1 >= 0 && excl + q0 < rem && rem <= excl + q0 + q1) {
        sm.found_bin = d1;
        sm.above_mass = count_mode ? excl_o + o0 : excl + q0;
        sm.above_cnt = count_mode ? excl + q0 : excl_o + o0;
      }
      if (rem == 0 && tid == 0) {  // gamma >= 1: nothing to find
        sm.found_bin = 0;
        sm.above_mass = 0;
        sm.above_cnt = 0;
      }
    }
    __syncthreads();
    {
      // this CTA's slice counts above the chosen digit (and, last pass, equal to
      // it) from its own histogram: elements > lambda / == lambda in the slice
      const uint32_t B = sm.found_bin;
      uint64_t part = 0;
      if (d0 >= 0 && (uint32_t)d0 > B) part += sm.cnt[d0];
      if (d1 >= 0 && (uint32_t)d1 > B) part += sm.cnt[d1];
      uint64_t tot_gt;
      block_scan_u64(part, sm.wsum, &tot_gt);
      slice_gt += tot_gt;
      if (pass == 2) slice_eq = sm.cnt[B];
    }
    prefix |= sm.found_bin << sh;
    pmask |= dmask << sh;
    above_mass_tot += sm.above_mass;
    above_cnt_tot += sm.above_cnt;
    rem -= count_mode ? sm.above_cnt : sm.above_mass;
    __syncthreads();
    FP_TM(4 + 4 * pass);
  }
  if (gamma >= 1.0f) {  // A7: everything, in index order
    for (long long i = lo + tid; i < hi; i += kSelThreads) out[i] = (int32_t)i;
    if (tid == 0 && sub == 0) {
      *count_out = (int32_t)L;
      *mass_out = T;
    }
    if (nr > 1) {
      cl_sync();  // keep the barrier count equal to the gamma < 1 path
      cl_sync();
    }
    return;
  }
  // lambda = prefix; take t of its ties (lowest indices first)
  const uint32_t lam = prefix;
  const uint64_t f_lam = fixp(__uint_as_float(lam));
  const uint64_t t_take = count_mode ? rem : (rem + f_lam - 1) / f_lam;
  const uint64_t K = above_cnt_tot + t_take;

  // slice counts (> lambda, == lambda), exchanged across the sub-group for the offsets
  if (tid == 0) {
    sm.slice_gt = slice_gt;
    sm.slice_eq = slice_eq;
  }
  uint64_t gt_run = 0, eq_run = 0;
  if (nr > 1) {
    cl_sync();
    for (uint32_t r = 0; r < sub; ++r) {
      gt_run += cl_ld64(cl_map(&sm.slice_gt, r0 + r));
      eq_run += cl_ld64(cl_map(&sm.slice_eq, r0 + r));
    }
  }
  FP_TM(13);
  // ordered compaction of this slice: the <= 3 keys before the first 16-B
  // boundary by thread 0, then a contiguous range per thread from that boundary
  const long long xmis = (long long)((reinterpret_cast<uintptr_t>(x) >> 2) & 3);
  const long long a0 = min(hi, lo + ((-(xmis + lo)) & 3));
  if (a0 > lo) {
    if (tid == 0) {
      uint64_t g = gt_run, q = eq_run;
      for (long long i = lo; i < a0; ++i) {
        const uint32_t key = __float_as_uint(__ldg(x + i));
        if (key > lam) {
          out[g + min(t_take, q)] = (int32_t)i;
          ++g;
        } else if (key == lam) {
          if (q < t_take) out[g + q] = (int32_t)i;
          ++q;
        }
      }
      sm.above_cnt = g;  // free after the passes: broadcast slots
      sm.above_mass = q;
    }
    __syncthreads();
    gt_run = sm.above_cnt;
    eq_run = sm.above_mass;
    __syncthreads();
  }
  // thread t owns the keys [a0 + t P, a0 + (t + 1) P) (P a multiple of 4:
  // 16-B loads): one pass counts its keys > lambda / == lambda, ONE block scan
  // gives every thread its output offset, a second pass over the same keys
  // (L1 / L2 resident) writes the selected indices in index order. (Rounds of
  // 8 consecutive keys per thread with a scan each -- also with the output
  // staged in shared memory for coalesced stores -- and four loads in flight
  // per thread here measured slower: profiles/r02s3_topmass_phases.txt.)
  const long long P = 4 * ((hi - a0 + 4LL * kSelThreads - 1) / (4LL * kSelThreads));
  const long long b0 = min(hi, a0 + (long long)tid * P), b1 = min(hi, b0 + P);
  auto load4 = [&](long long i, uint32_t* kk) {
    if (i + 4 <= b1) {
      const float4 f4 = __ldg(reinterpret_cast<const float4*>(x + i));
      kk[0] = __float_as_uint(f4.x);
      kk[1] = __float_as_uint(f4.y);
      kk[2] = __float_as_uint(f4.z);
      kk[3] = __float_as_uint(f4.w);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) kk[e] = i + e < b1 ? __float_as_uint(__ldg(x + i + e)) : 0u;
    }
  };
  uint32_t gt = 0, eq = 0;
  for (long long i = b0; i < b1; i += 4) {
    uint32_t kk[4];
    load4(i, kk);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const bool valid = i + e < b1;
      gt += (valid && kk[e] > lam);
      eq += (valid && kk[e] == lam);
    }
  }
  {
    uint64_t tot;
    const uint64_t packed = ((uint64_t)eq << 32) | gt;
    const uint64_t excl = block_scan_u64(packed, sm.wsum, &tot) - packed;
    uint64_t eq_pre = eq_run + (excl >> 32);
    uint64_t pos = gt_run + (excl & 0xffffffffu) + min(t_take, eq_pre);
    for (long long i = b0; i < b1; i += 4) {
      uint32_t kk[4];
      load4(i, kk);
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (i + e >= b1) break;
        bool take = kk[e] > lam;
        if (kk[e] == lam) {
          take = eq_pre < t_take;
          ++eq_pre;
        }
        if (take) out[pos++] = (int32_t)(i + e);
      }
    }
  }
  FP_TM(14);
  if (tid == 0 && sub == 0) {
    *count_out = (int32_t)K;
    *mass_out = above_mass_tot + t_take * f_lam;
  }
  if (nr > 1) cl_sync();  // keep this CTA's shared memory alive until the sub-group is done
  FP_TM(15);
}

// One cluster of C CTAs (1, 2, 4 or 8; set at launch) per head. VS head:
// ranks [0, C/2) select the vertical lines (a_v, or a_hat with vs_mode 1),
// ranks [C/2, C) the slash lines (a_s, or As) -- with C = 1 the one CTA does
// both, one after the other. QA head: all C ranks on the flattened map.
__global__ void __launch_bounds__(kSelThreads, 1)
    topmass_kernel(const float* __restrict__ a_v, const float* __restrict__ a_s,
                   const float* __restrict__ a_hat, const float* __restrict__ As,
                   const float* __restrict__ A_bar, const int32_t* __restrict__ pattern, int n,
                   int nb, long long tri, float gamma, int vs_mode, int qa_mode,
                   int32_t* __restrict__ sel_v, int32_t* __restrict__ sel_s,
                   int32_t* __restrict__ sel_qa, int32_t* __restrict__ sel_count,
                   unsigned long long* __restrict__ sel_mass) {
  FP_PDL_ENTRY();
  extern __shared__ __align__(16) uint8_t top_raw[];
  TopSmem& sm = *reinterpret_cast<TopSmem*>(top_raw);
  uint32_t ncl;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncl));
  const int h = blockIdx.y;
  const uint32_t crank = cl_rank();
  const int tid = threadIdx.x;
  const int pat = pattern[h];
  if (pat == 1) {
    if (tid == 0 && crank == 0) {
      for (int sg = 0; sg < 2; ++sg) {
        sel_count[h * 4 + sg] = 0;
        sel_mass[h * 4 + sg] = 0;
      }
    }
    if (qa_mode == 1) {  // per-row QA selection is topmass_rows: the cluster leaves together
      if (tid == 0 && crank == 0) {
        sel_count[h * 4 + 2] = 0;
        sel_mass[h * 4 + 2] = 0;
      }
      return;
    }
    topmass_segment(sm, A_bar + (size_t)h * tri, tri, sel_qa + (size_t)h * tri, gamma, 0, ncl, crank,
                    &sel_count[h * 4 + 2], &sel_mass[h * 4 + 2]);
    return;
  }
  if (tid == 0 && crank == 0) {
    sel_count[h * 4 + 2] = 0;
    sel_mass[h * 4 + 2] = 0;
  }
  const long long L = vs_mode ? nb : n;
  const float* xv = vs_mode ? a_hat + (size_t)h * nb : a_v + (size_t)h * n;
  const float* xs = vs_mode ? As + (size_t)h * nb : a_s + (size_t)h * n;
  if (ncl == 1) {
    topmass_segment(sm, xv, L, sel_v + (size_t)h * n, gamma, 0, 1, 0, &sel_count[h * 4 + 0],
                    &sel_mass[h * 4 + 0]);
    __syncthreads();
    topmass_segment(sm, xs, L, sel_s + (size_t)h * n, gamma, 0, 1, 0, &sel_count[h * 4 + 1],
                    &sel_mass[h * 4 + 1]);
    return;
  }
  const uint32_t half = ncl / 2;
  const int seg = crank < half ? 0 : 1;
  topmass_segment(sm, seg == 0 ? xv : xs, L, (seg == 0 ? sel_v : sel_s) + (size_t)h * n, gamma,
                  seg * half, half, crank - seg * half, &sel_count[h * 4 + seg], &sel_mass[h * 4 + seg]);
}

// ---------------------------------------------------------------------------
// f2 (qa_mode 1, "wo/ flatten"): topmass of each row of A_bar, one
// CTA of 256 threads per (query block, QA head); same radix select by mass as
// topmass_kernel (fixed point, ties -> lower kb), output as a row bitmap.
constexpr int kRowThreads = 256;
struct RowSmem {
  uint32_t cnt[2048];
  unsigned long long mass[2048];
  uint64_t wsum[32];
  uint32_t bits[256];  // nb <= 8192 -> 256 words
  uint32_t found_bin;
  unsigned long long above_mass, above_cnt;
};

__device__ uint64_t block_scan_u64_256(uint64_t v, uint64_t* wsum, uint64_t* total) {
  const int ln = lane_id(), w = warp_id();
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint64_t y = __shfl_up_sync(0xffffffffu, v, o);
    if (ln >= o) v += y;
  }
  if (ln == 31) wsum[w] = v;
  __syncthreads();
  if (w == 0) {
    uint64_t s = (ln < kRowThreads / 32) ? wsum[ln] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (ln >= o) s += y;
    }
    if (ln < kRowThreads / 32) wsum[ln] = s;
  }
  __syncthreads();
  const uint64_t add = (w > 0) ? wsum[w - 1] : 0;
  const uint64_t tot = wsum[kRowThreads / 32 - 1];
  __syncthreads();
  *total = tot;
  return v + add;
}

__global__ void __launch_bounds__(kRowThreads) topmass_rows(
    const float* __restrict__ A_bar, const int32_t* __restrict__ pattern, int nb, int nbw,
    long long tri, float gamma, uint32_t* __restrict__ selbits, int32_t* __restrict__ sel_count,
    unsigned long long* __restrict__ sel_mass) {
  FP_PDL_ENTRY();
  __shared__ RowSmem sm;
  const int qb = blockIdx.x, h = blockIdx.y;
  if (pattern[h] != 1) return;
  const float* x = A_bar + (size_t)h * tri + (size_t)qb * (qb + 1) / 2;
  const int L = qb + 1;
  const int tid = threadIdx.x;
  for (int i = tid; i < nbw; i += kRowThreads) sm.bits[i] = 0;
  unsigned long long T = 0, rem = 0, K = 0, mass_sel = 0;
  bool count_mode = false, all = false;
  uint32_t prefix = 0, pmask = 0;
  unsigned long long above_mass_tot = 0, above_cnt_tot = 0;
  const int shifts[3] = {21, 10, 0};
  const int widths[3] = {11, 11, 10};
  for (int pass = 0; pass < 3 && !all; ++pass) {
    const int sh = shifts[pass];
    const uint32_t dmask = (1u << widths[pass]) - 1u;
    const int nbins = 1 << widths[pass];
    for (int b = tid; b < 2048; b += kRowThreads) {
      sm.cnt[b] = 0;
      sm.mass[b] = 0;
    }
    __syncthreads();
    for (int base = 0; base < L; base += kRowThreads) {
      const int i = base + tid;
      const bool valid = i < L;
      const uint32_t key = valid ? __float_as_uint(x[i]) : 0xffffffffu;
      const bool match = valid && ((key & pmask) == prefix);
      const uint32_t digit = match ? ((key >> sh) & dmask) : 0xffffffffu;
      const uint32_t grp = __match_any_sync(0xffffffffu, digit);
      if (match) {
        const uint64_t f = fixp(__uint_as_float(key));
        const uint32_t s0 = __reduce_add_sync(grp, (uint32_t)(f & 0xFFFFF));
        const uint32_t s1 = __reduce_add_sync(grp, (uint32_t)((f >> 20) & 0xFFFFF));
        const uint32_t s2 = __reduce_add_sync(grp, (uint32_t)(f >> 40));
        if ((__ffs(grp) - 1) == (int)lane_id()) {
          atomicAdd(&sm.cnt[digit], (uint32_t)__popc(grp));
          atomicAdd(&sm.mass[digit], ((unsigned long long)s2 << 40) +
                                         ((unsigned long long)s1 << 20) + (unsigned long long)s0);
        }
      }
    }
    __syncthreads();
    // thread t owns the 8 digits nbins-1-8t .. nbins-8-8t (descending)
    uint64_t km[8], kc[8], pm = 0, pc = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int d = nbins - 1 - 8 * tid - j;
      km[j] = (d >= 0) ? sm.mass[d] : 0;
      kc[j] = (d >= 0) ? sm.cnt[d] : 0;
      pm += km[j];
      pc += kc[j];
    }
    uint64_t tot_m, tot_c;
    uint64_t excl_m = block_scan_u64_256(pm, sm.wsum, &tot_m) - pm;
    uint64_t excl_c = block_scan_u64_256(pc, sm.wsum, &tot_c) - pc;
    if (pass == 0) {
      T = tot_m;
      if (gamma >= 1.0f) {  // A7: everything
        all = true;
        K = L;
        mass_sel = T;
        break;
      }
      const unsigned long long G = (unsigned long long)ceil((double)gamma * (double)T);
      count_mode = (G == 0);
      rem = count_mode ? 1ull : G;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const uint64_t q = count_mode ? kc[j] : km[j];
      const uint64_t e = count_mode ? excl_c : excl_m;
      if (nbins - 1 - 8 * tid - j >= 0 && e < rem && rem <= e + q) {
        sm.found_bin = nbins - 1 - 8 * tid - j;
        sm.above_mass = excl_m;
        sm.above_cnt = excl_c;
      }
      excl_m += km[j];
      excl_c += kc[j];
    }
    __syncthreads();
    prefix |= sm.found_bin << sh;
    pmask |= dmask << sh;
    above_mass_tot += sm.above_mass;
    above_cnt_tot += sm.above_cnt;
    rem -= count_mode ? sm.above_cnt : sm.above_mass;
    __syncthreads();
  }
  uint32_t lam = prefix;
  uint64_t t_take = 0;
  if (!all) {
    const uint64_t f_lam = fixp(__uint_as_float(lam));
    t_take = count_mode ? rem : (rem + f_lam - 1) / f_lam;
    K = above_cnt_tot + t_take;
    mass_sel = above_mass_tot + t_take * f_lam;
  }
  // selection bits in index order (ties: the first t_take occurrences of lambda)
  uint64_t eq_run = 0;
  for (int base = 0; base < L; base += kRowThreads) {
    const int i = base + tid;
    const bool valid = i < L;
    const uint32_t key = valid ? __float_as_uint(x[i]) : 0u;
    const bool eq = valid && !all && key == lam;
    uint64_t tot;
    const uint64_t excl = block_scan_u64_256(eq ? 1 : 0, sm.wsum, &tot) - (eq ? 1 : 0);
    const bool take = valid && (all || key > lam || (eq && eq_run + excl < t_take));
    if (take) atomicOr(&sm.bits[i >> 5], 1u << (i & 31));
    eq_run += tot;
  }
  __syncthreads();
  uint32_t* dst = selbits + ((size_t)h * nb + qb) * nbw;
  for (int i = tid; i < nbw; i += kRowThreads) dst[i] = sm.bits[i];
  if (tid == 0) {
    atomicAdd(&sel_count[h * 4 + 2], (int32_t)K);
    atomicAdd(&sel_mass[h * 4 + 2], mass_sel);
  }
}

// vertical-block and slash-diagonal bitmaps of VS heads (A10, reading R1):
// V / Dg are this CTA's shared-memory bitmaps (nbw words each), also stored
// to vbits / dbits. All threads of the CTA call it.
__device__ void build_lines_body(int h, uint32_t* V, uint32_t* Dg, const int32_t* __restrict__ pattern,
                                 const int32_t* __restrict__ sel_v, const int32_t* __restrict__ sel_s,
                                 const int32_t* __restrict__ sel_count, int n, int nb, int nbw, int vs_mode,
                                 int lb, uint32_t* __restrict__ vbits, uint32_t* __restrict__ dbits) {
  for (int w = threadIdx.x; w < nbw; w += blockDim.x) V[w] = Dg[w] = 0;
  __syncthreads();
  if (pattern[h] == 0) {
    const int kv = sel_count[h * 4 + 0], ks = sel_count[h * 4 + 1];
    const int32_t* sv = sel_v + (size_t)h * n;
    const int32_t* ss = sel_s + (size_t)h * n;
    for (int i = threadIdx.x; i < kv; i += blockDim.x) {
      const int kb = vs_mode ? sv[i] : (sv[i] >> lb);
      atomicOr(&V[kb >> 5], 1u << (kb & 31));
    }
    for (int i = threadIdx.x; i < ks; i += blockDim.x) {
      const int o = ss[i];
      const int d = vs_mode ? o : (o >> lb);
      atomicOr(&Dg[d >> 5], 1u << (d & 31));
      // R1: offset o crosses diagonals o/b and o/b + 1 (unless aligned);
      // R2 (vs_mode 1): the offset group [d b, (d+1) b) covers d and d + 1
      if ((vs_mode || (o & ((1 << lb) - 1))) && d + 1 < nb) atomicOr(&Dg[(d + 1) >> 5], 1u << ((d + 1) & 31));
    }
  }
  __syncthreads();
  for (int w = threadIdx.x; w < nbw; w += blockDim.x) {
    vbits[(size_t)h * nbw + w] = V[w];
    dbits[(size_t)h * nbw + w] = Dg[w];
  }
}
__global__ void build_lines(const int32_t* __restrict__ pattern, const int32_t* __restrict__ sel_v,
                            const int32_t* __restrict__ sel_s, const int32_t* __restrict__ sel_count,
                            int n, int nb, int nbw, int vs_mode, int lb, uint32_t* __restrict__ vbits,
                            uint32_t* __restrict__ dbits) {
  FP_PDL_ENTRY();
  extern __shared__ uint32_t bsm[];  // V[nbw] | D[nbw]
  build_lines_body(blockIdx.x, bsm, bsm + nbw, pattern, sel_v, sel_s, sel_count, n, nb, nbw, vs_mode, lb,
                   vbits, dbits);
}

__device__ __forceinline__ bool bit_at(const uint32_t* b, int i) { return (b[i >> 5] >> (i & 31)) & 1u; }

// one warp per (head, query-block row)
constexpr int kAsmWarps = 8;
// One query-block row qb of head h, by one warp: rasterised lines or QA
// blocks, forced blocks (A11), minimum / maximum budget (A12, A23); row / keep
// are the warp's nbw-word scratch, V / Dg the head's line bitmaps.
__device__ void assemble_row(int h, int qb, uint32_t* row, uint32_t* keep, const uint32_t* V,
                             const uint32_t* Dg, const int32_t* __restrict__ pattern,
                             const int32_t* __restrict__ sel_qa, const int32_t* __restrict__ sel_count,
                             const float* __restrict__ a_hat, const float* __restrict__ As,
                             const float* __restrict__ A_bar, int nb, int nbw, long long tri, int min_blocks,
                             int qa_mode, const uint32_t* __restrict__ selbits, int max_blocks,
                             uint32_t* __restrict__ rowbits, int32_t* __restrict__ row_nnz,
                             int32_t* __restrict__ row_nnz_pre, int32_t* __restrict__ budget_added,
                             int32_t* __restrict__ budget_removed) {
  const int ln = lane_id();
  const int pat = pattern[h];
  for (int i = ln; i < nbw; i += 32) row[i] = 0;
  __syncwarp();
  const int nw_row = (qb >> 5) + 1;  // words that can hold kb <= qb
  if (pat == 0) {
    for (int wd = 0; wd < nw_row; ++wd) {
      const int kb = wd * 32 + ln;
      const bool on = (kb <= qb) && (bit_at(V, kb) || bit_at(Dg, qb - kb));
      const uint32_t word = __ballot_sync(0xffffffffu, on);
      if (ln == 0) row[wd] = word;
    }
  } else if (qa_mode == 1) {
    // per-row selection already as a bitmap (topmass_rows)
    const uint32_t* src = selbits + ((size_t)h * nb + qb) * nbw;
    for (int i = ln; i < nw_row; i += 32) row[i] = src[i];
  } else {
    // S_qa is sorted; this row's flat indices are [qb(qb+1)/2, qb(qb+1)/2 + qb]
    const int kq = sel_count[h * 4 + 2];
    const int32_t* sq = sel_qa + (size_t)h * tri;
    const long long lo = (long long)qb * (qb + 1) / 2, hi = lo + qb;
    // lower bound of lo (every lane does the same binary search)
    int a = 0, b = kq;
    while (a < b) {
      const int mid = (a + b) >> 1;
      if (sq[mid] < lo) a = mid + 1; else b = mid;
    }
    for (int i = a + ln; i < kq; i += 32) {
      const long long p = sq[i];
      if (p > hi) break;
      const int kb = (int)(p - lo);
      atomicOr(&row[kb >> 5], 1u << (kb & 31));
    }
  }
  __syncwarp();
  if (ln == 0) {
    row[0] |= 1u;                       // first key block (A11)
    row[qb >> 5] |= 1u << (qb & 31);    // diagonal = last key block of the row
  }
  __syncwarp();
  int cnt = 0;
  for (int wd = ln; wd < nw_row; wd += 32) cnt += __popc(row[wd]);
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  const int pre = cnt;
  // minimum budget (A12): best unselected kb <= qb by row score, ties -> lower kb
  const int need = min(min_blocks, qb + 1) - cnt;
  const float* Ab = A_bar + (size_t)h * tri + (size_t)qb * (qb + 1) / 2;
  for (int it = 0; it < need; ++it) {
    float best = -INFINITY;
    int bkb = 0x7fffffff;
    for (int kb = ln; kb <= qb; kb += 32) {
      if (bit_at(row, kb)) continue;
      const float sc = (pat == 0) ? __fadd_rn(a_hat[(size_t)h * nb + kb], As[(size_t)h * nb + qb - kb])
                                  : Ab[kb];
      if (sc > best || (sc == best && kb < bkb)) {
        best = sc;
        bkb = kb;
      }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const float ob = __shfl_xor_sync(0xffffffffu, best, o);
      const int ok = __shfl_xor_sync(0xffffffffu, bkb, o);
      if (ob > best || (ob == best && ok < bkb)) {
        best = ob;
        bkb = ok;
      }
    }
    if (ln == 0) row[bkb >> 5] |= 1u << (bkb & 31);
    __syncwarp();
  }
  const int added = need > 0 ? need : 0;
  // maximum budget (A23): rows above the cap keep the forced blocks and the
  // best remaining selected blocks by row score (ties -> lower kb)
  int removed = 0;
  const int nforced = (qb == 0) ? 1 : 2;
  const int cap = max(max_blocks, nforced);
  if (max_blocks > 0 && pre + added > cap) {
    for (int i = ln; i < nbw; i += 32) keep[i] = 0;
    __syncwarp();
    if (ln == 0) {
      keep[0] |= 1u;
      keep[qb >> 5] |= 1u << (qb & 31);
    }
    __syncwarp();
    for (int it = 0; it < cap - nforced; ++it) {
      float best = -INFINITY;
      int bkb = 0x7fffffff;
      for (int kb = ln; kb <= qb; kb += 32) {
        if (!bit_at(row, kb) || bit_at(keep, kb)) continue;
        const float sc = (pat == 0) ? __fadd_rn(a_hat[(size_t)h * nb + kb], As[(size_t)h * nb + qb - kb])
                                    : Ab[kb];
        if (sc > best || (sc == best && kb < bkb)) {
          best = sc;
          bkb = kb;
        }
      }
      for (int o = 16; o > 0; o >>= 1) {
        const float ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int ok = __shfl_xor_sync(0xffffffffu, bkb, o);
        if (ob > best || (ob == best && ok < bkb)) {
          best = ob;
          bkb = ok;
        }
      }
      if (ln == 0) keep[bkb >> 5] |= 1u << (bkb & 31);
      __syncwarp();
    }
    for (int i = ln; i < nbw; i += 32) row[i] = keep[i];
    __syncwarp();
    removed = pre + added - cap;
  }
  uint32_t* dst = rowbits + ((size_t)h * nb + qb) * nbw;
  for (int i = ln; i < nbw; i += 32) dst[i] = row[i];
  if (ln == 0) {
    row_nnz[(size_t)h * nb + qb] = pre + added - removed;
    row_nnz_pre[(size_t)h * nb + qb] = pre;
    budget_added[(size_t)h * nb + qb] = added;
    budget_removed[(size_t)h * nb + qb] = removed;
  }
}

__global__ void __launch_bounds__(kAsmWarps * 32) assemble_rows(
    const int32_t* __restrict__ pattern, const uint32_t* __restrict__ vbits,
    const uint32_t* __restrict__ dbits, const int32_t* __restrict__ sel_qa,
    const int32_t* __restrict__ sel_count, const float* __restrict__ a_hat,
    const float* __restrict__ As, const float* __restrict__ A_bar, int nb, int nbw,
    long long tri, int min_blocks, int qa_mode, const uint32_t* __restrict__ selbits,
    int max_blocks, uint32_t* __restrict__ rowbits, int32_t* __restrict__ row_nnz,
    int32_t* __restrict__ row_nnz_pre, int32_t* __restrict__ budget_added,
    int32_t* __restrict__ budget_removed) {
  FP_PDL_ENTRY();
  extern __shared__ uint32_t asmem[];  // [kAsmWarps][2][nbw]
  const int h = blockIdx.y;
  const int w = warp_id();
  const int qb = blockIdx.x * kAsmWarps + w;
  if (qb >= nb) return;
  uint32_t* row = asmem + w * 2 * nbw;
  assemble_row(h, qb, row, row + nbw, vbits + (size_t)h * nbw, dbits + (size_t)h * nbw, pattern, sel_qa,
               sel_count, a_hat, As, A_bar, nb, nbw, tri, min_blocks, qa_mode, selbits, max_blocks, rowbits,
               row_nnz, row_nnz_pre, budget_added, budget_removed);
}

// exclusive scan of row nnz per head -> row_ptr; stats
// exclusive scan of row nnz of head h -> row_ptr; stats (all threads of a
// kSelThreads CTA; wsum: 32 words of shared scratch)
__device__ void row_scan_body(int h, uint64_t* wsum, const int32_t* __restrict__ row_nnz,
                              const int32_t* __restrict__ budget_added,
                              const int32_t* __restrict__ budget_removed, const int32_t* __restrict__ pattern,
                              const int32_t* __restrict__ sel_count,
                              const unsigned long long* __restrict__ sel_mass, int nb,
                              int32_t* __restrict__ row_ptr, fp_select_stats* __restrict__ stats) {
  uint64_t run = 0, badd = 0, brem = 0;
  for (int base = 0; base < nb; base += kSelThreads) {
    const int i = base + threadIdx.x;
    const uint64_t v = (i < nb) ? (uint64_t)row_nnz[(size_t)h * nb + i] : 0;
    const uint64_t ba = (i < nb) ? (uint64_t)budget_added[(size_t)h * nb + i] : 0;
    const uint64_t br = (i < nb) ? (uint64_t)budget_removed[(size_t)h * nb + i] : 0;
    uint64_t tot, tot2;
    const uint64_t packed = (ba << 32) | v;
    const uint64_t incl = block_scan_u64(packed, wsum, &tot);
    block_scan_u64(br, wsum, &tot2);
    if (i < nb) row_ptr[(size_t)h * (nb + 1) + i] = (int32_t)(run + ((incl - packed) & 0xffffffffu));
    run += tot & 0xffffffffu;
    badd += tot >> 32;
    brem += tot2;
  }
  if (threadIdx.x == 0) {
    row_ptr[(size_t)h * (nb + 1) + nb] = (int32_t)run;
    if (stats) {
      fp_select_stats st;
      const double inv = 1.0 / 1152921504606846976.0;
      st.pattern = pattern[h];
      st.k_v = sel_count[h * 4 + 0];
      st.k_s = sel_count[h * 4 + 1];
      st.k_qa = sel_count[h * 4 + 2];
      st.mass_v = (double)sel_mass[h * 4 + 0] * inv;
      st.mass_s = (double)sel_mass[h * 4 + 1] * inv;
      st.mass_qa = (double)sel_mass[h * 4 + 2] * inv;
      st.nnz_blocks = (int32_t)run;
      st.budget_added = (int32_t)badd;
      st.budget_removed = (int32_t)brem;
      stats[h] = st;
    }
  }
}

__global__ void __launch_bounds__(kSelThreads, 1)
    row_scan(const int32_t* __restrict__ row_nnz, const int32_t* __restrict__ budget_added,
             const int32_t* __restrict__ budget_removed,
             const int32_t* __restrict__ pattern, const int32_t* __restrict__ sel_count,
             const unsigned long long* __restrict__ sel_mass, int nb, int32_t* __restrict__ row_ptr,
             fp_select_stats* __restrict__ stats) {
  FP_PDL_ENTRY();
  __shared__ uint64_t wsum[32];
  row_scan_body(blockIdx.x, wsum, row_nnz, budget_added, budget_removed, pattern, sel_count, sel_mass, nb,
                row_ptr, stats);
}

// the CSR column indices of row qb of head h (ascending kb), by one warp
__device__ void write_row(int h, int qb, const uint32_t* __restrict__ rowbits, const int32_t* __restrict__ row_ptr,
                          int nb, int nbw, long long cap, int32_t* __restrict__ col_idx) {
  const int ln = lane_id();
  const uint32_t* row = rowbits + ((size_t)h * nb + qb) * nbw;
  int32_t* out = col_idx + (size_t)h * cap + row_ptr[(size_t)h * (nb + 1) + qb];
  int pos = 0;
  const int nw_row = (qb >> 5) + 1;
  for (int wd = 0; wd < nw_row; ++wd) {
    const uint32_t word = row[wd];
    if ((word >> ln) & 1u) out[pos + __popc(word & ((1u << ln) - 1u))] = wd * 32 + ln;
    pos += __popc(word);
  }
}
__global__ void __launch_bounds__(kAsmWarps * 32) write_cols(
    const uint32_t* __restrict__ rowbits, const int32_t* __restrict__ row_ptr, int nb, int nbw,
    long long cap, int32_t* __restrict__ col_idx) {
  FP_PDL_ENTRY();
  const int h = blockIdx.y;
  const int qb = blockIdx.x * kAsmWarps + warp_id();
  if (qb >= nb) return;
  write_row(h, qb, rowbits, row_ptr, nb, nbw, cap, col_idx);
}

// Short sequences (nb <= kPostSmallNb): lines, rows, scan and columns of one
// head in ONE CTA of kSelThreads (32 warps, each a stripe of rows) -- the same
// device code as the four kernels above, so the same CSR, in one launch
// instead of four (each of which costs its launch / ramp at this size).
constexpr int kPostSmallNb = 64;
__global__ void __launch_bounds__(kSelThreads, 1) select_post_small(
    const int32_t* __restrict__ pattern, const int32_t* __restrict__ sel_v, const int32_t* __restrict__ sel_s,
    const int32_t* __restrict__ sel_qa, const int32_t* __restrict__ sel_count,
    const unsigned long long* __restrict__ sel_mass, const float* __restrict__ a_hat,
    const float* __restrict__ As, const float* __restrict__ A_bar, int n, int nb, int nbw, long long tri,
    int vs_mode, int lb, int min_blocks, int qa_mode, const uint32_t* __restrict__ selbits, int max_blocks,
    uint32_t* __restrict__ vbits, uint32_t* __restrict__ dbits, uint32_t* __restrict__ rowbits,
    int32_t* __restrict__ row_nnz, int32_t* __restrict__ row_nnz_pre, int32_t* __restrict__ budget_added,
    int32_t* __restrict__ budget_removed, int32_t* __restrict__ row_ptr, fp_select_stats* __restrict__ stats,
    int32_t* __restrict__ col_idx) {
  FP_PDL_ENTRY();
  __shared__ uint32_t V[kPostSmallNb / 32], Dg[kPostSmallNb / 32];
  __shared__ uint32_t scr[kSelThreads / 32][2][kPostSmallNb / 32];
  __shared__ uint64_t wsum[32];
  const int h = blockIdx.x;
  const int w = warp_id();
  build_lines_body(h, V, Dg, pattern, sel_v, sel_s, sel_count, n, nb, nbw, vs_mode, lb, vbits, dbits);
  __syncthreads();
  for (int qb = w; qb < nb; qb += kSelThreads / 32)
    assemble_row(h, qb, scr[w][0], scr[w][1], V, Dg, pattern, sel_qa, sel_count, a_hat, As, A_bar, nb, nbw,
                 tri, min_blocks, qa_mode, selbits, max_blocks, rowbits, row_nnz, row_nnz_pre, budget_added,
                 budget_removed);
  __syncthreads();
  row_scan_body(h, wsum, row_nnz, budget_added, budget_removed, pattern, sel_count, sel_mass, nb, row_ptr,
                stats);
  __syncthreads();
  for (int qb = w; qb < nb; qb += kSelThreads / 32) write_row(h, qb, rowbits, row_ptr, nb, nbw, tri, col_idx);
}

}  // namespace

cudaError_t launch_select(const Shape& s, const WsLayout& L, void* ws, float gamma, int min_budget,
                          const fp_select_options& opt, int32_t* row_ptr, int32_t* col_idx,
                          fp_select_stats* stats, cudaStream_t st) {
  const int32_t* pat = wsp<int32_t>(ws, L.pattern);
  const cudaError_t ea = ensure_smem_attr((const void*)topmass_kernel, sizeof(TopSmem));
  if (ea != cudaSuccess) return ea;
  {
    // cluster size per head: <= ~160K scores per CTA for the flattened QA map,
    // <= ~80K per CTA for each of the two VS segments (C/2 CTAs each), 1..8 CTAs
    const long long lvs = opt.vs_mode ? s.nb : s.n, lqa = opt.qa_mode ? 0 : s.tri;
    long long need = std::max((lqa + 159999) / 160000, 2 * ((lvs + 79999) / 80000));
    int ncl = 1;
    while (ncl < need && ncl < kClMax) ncl <<= 1;
    // more CTAs per head while the whole grid still fits in one wave (one
    // 1024-thread CTA per SM) and a VS CTA keeps >= kTopMinKeys scores: the
    // histogram passes scale with the slice, the barriers and scans do not
    {
      int nsm = 148, dev = 0;
      if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
      // (a VS segment gets ncl / 2 CTAs: after doubling, lvs / ncl scores each)
      while (ncl < kClMax && (long long)s.H * ncl * 2 <= nsm && lvs / ncl >= kTopMinKeys) ncl <<= 1;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ncl, s.H);
    cfg.blockDim = dim3(kSelThreads);
    cfg.dynamicSmemBytes = sizeof(TopSmem);
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ncl;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // PDL (FP_PDL_ENTRY)
#ifdef FP_NO_PDL
    attr[1].val.programmaticStreamSerializationAllowed = 0;
#else
    attr[1].val.programmaticStreamSerializationAllowed = 1;
#endif
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    cudaError_t e = cudaLaunchKernelEx(
        &cfg, topmass_kernel, (const float*)wsp<float>(ws, L.a_v), (const float*)wsp<float>(ws, L.a_s),
        (const float*)wsp<float>(ws, L.a_hat), (const float*)wsp<float>(ws, L.As),
        (const float*)wsp<float>(ws, L.A_bar), pat, s.n, s.nb, s.tri, gamma, (int)opt.vs_mode,
        (int)opt.qa_mode, wsp<int32_t>(ws, L.sel_v), wsp<int32_t>(ws, L.sel_s),
        wsp<int32_t>(ws, L.sel_qa), wsp<int32_t>(ws, L.sel_count),
        wsp<unsigned long long>(ws, L.sel_mass));
    if (e != cudaSuccess) return e;
  }
  if (opt.qa_mode == 1)
    FP_LAUNCH(topmass_rows, dim3(s.nb, s.H), kRowThreads, 0, st, 
        wsp<float>(ws, L.A_bar), pat, s.nb, L.nbw, s.tri, gamma, wsp<uint32_t>(ws, L.selbits),
        wsp<int32_t>(ws, L.sel_count), wsp<unsigned long long>(ws, L.sel_mass));
  // A12 / f2: budgets in tokens -> key blocks of this block size
  // (int64: token budgets near INT_MAX must not overflow; clamped to nb)
  const int min_blocks = (int)std::min<long long>(s.nb, ((long long)min_budget + s.b - 1) / s.b);
  const int max_blocks = (int)std::min<long long>(s.nb, ((long long)opt.max_budget + s.b - 1) / s.b);
  if (s.nb <= kPostSmallNb) {
    FP_LAUNCH(select_post_small, s.H, kSelThreads, 0, st, pat, wsp<int32_t>(ws, L.sel_v), wsp<int32_t>(ws, L.sel_s),
              wsp<int32_t>(ws, L.sel_qa), wsp<int32_t>(ws, L.sel_count), wsp<unsigned long long>(ws, L.sel_mass),
              wsp<float>(ws, L.a_hat), wsp<float>(ws, L.As), wsp<float>(ws, L.A_bar), s.n, s.nb, L.nbw, s.tri,
              opt.vs_mode, s.lb, min_blocks, opt.qa_mode, wsp<uint32_t>(ws, L.selbits), max_blocks,
              wsp<uint32_t>(ws, L.vbits), wsp<uint32_t>(ws, L.dbits), wsp<uint32_t>(ws, L.rowbits),
              wsp<int32_t>(ws, L.row_nnz), wsp<int32_t>(ws, L.row_nnz_pre), wsp<int32_t>(ws, L.budget_added),
              wsp<int32_t>(ws, L.budget_removed), row_ptr, stats, col_idx);
    return cudaGetLastError();
  }
  FP_LAUNCH(build_lines, s.H, 1024, 2 * L.nbw * 4, st, pat, wsp<int32_t>(ws, L.sel_v),
                                                wsp<int32_t>(ws, L.sel_s),
                                                wsp<int32_t>(ws, L.sel_count), s.n, s.nb, L.nbw,
                                                opt.vs_mode, s.lb, wsp<uint32_t>(ws, L.vbits),
                                                wsp<uint32_t>(ws, L.dbits));
  const dim3 rg((s.nb + kAsmWarps - 1) / kAsmWarps, s.H);
  FP_LAUNCH(assemble_rows, rg, kAsmWarps * 32, kAsmWarps * 2 * L.nbw * 4, st, 
      pat, wsp<uint32_t>(ws, L.vbits), wsp<uint32_t>(ws, L.dbits), wsp<int32_t>(ws, L.sel_qa),
      wsp<int32_t>(ws, L.sel_count), wsp<float>(ws, L.a_hat), wsp<float>(ws, L.As),
      wsp<float>(ws, L.A_bar), s.nb, L.nbw, s.tri, min_blocks, opt.qa_mode,
      wsp<uint32_t>(ws, L.selbits), max_blocks, wsp<uint32_t>(ws, L.rowbits),
      wsp<int32_t>(ws, L.row_nnz), wsp<int32_t>(ws, L.row_nnz_pre), wsp<int32_t>(ws, L.budget_added),
      wsp<int32_t>(ws, L.budget_removed));
  FP_LAUNCH(row_scan, s.H, kSelThreads, 0, st, wsp<int32_t>(ws, L.row_nnz), wsp<int32_t>(ws, L.budget_added),
                                        wsp<int32_t>(ws, L.budget_removed), pat,
                                        wsp<int32_t>(ws, L.sel_count),
                                        wsp<unsigned long long>(ws, L.sel_mass), s.nb, row_ptr, stats);
  FP_LAUNCH(write_cols, rg, kAsmWarps * 32, 0, st, wsp<uint32_t>(ws, L.rowbits), row_ptr, s.nb, L.nbw,
                                            s.tri, col_idx);
  return cudaGetLastError();
}

}  // namespace fp

#ifdef FP_TM_TIMING
extern "C" int fp_debug_topmass_timing(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, fp::g_tm_t, sizeof(fp::g_tm_t));
}
#endif
