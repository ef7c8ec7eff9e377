// Microbenchmark of tcgen05.mma kind::f16 on sm_100a: cycles per M=128 x N x
// K=16 MMA for A from shared memory (SS) or tensor memory (TS), with every
// descriptor precomputed (8-step unrolled issue loop) so that the issuing
// thread is not the limiter. One CTA per SM, one issuing thread.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#include "../paper_2502_20766_b200/csrc/fp_common.cuh"

using namespace fp;

constexpr int ITER = 256;  // x 8 MMAs

FP_DEV void umma_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(bdesc), "r"(idesc), "r"(acc));
}

// 8 MMAs in one asm statement (one elect/waterfall wrapper for all of them)
FP_DEV void umma_ts8(uint32_t d, uint32_t a0, const uint64_t* bd, uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 1, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %3, %11, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%2], %4, %11, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%12], %5, %11, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%13], %6, %11, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%14], %7, %11, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%15], %8, %11, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%16], %9, %11, p;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%17], %10, %11, p;\n\t}" ::"r"(d),
      "r"(a0), "r"(a0 + 8), "l"(bd[0]), "l"(bd[1]), "l"(bd[2]), "l"(bd[3]), "l"(bd[4]), "l"(bd[5]),
      "l"(bd[6]), "l"(bd[7]), "r"(idesc), "r"(a0 + 16), "r"(a0 + 24), "r"(a0 + 32), "r"(a0 + 40),
      "r"(a0 + 48), "r"(a0 + 56));
}

__device__ volatile int g_stop;
template <int MODE, int N, int ND, int LDW = 0, int CM = 0>
__global__ void __launch_bounds__(384, 1) kern(long long* out) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar, bar2[4];
  __shared__ uint32_t tbase_s;
  uint8_t* A = smem;          // 32 KiB
  uint8_t* B = smem + 32768;  // 64 KiB
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u;
  __shared__ volatile int stop;
  if (threadIdx.x == 0) stop = 0;
  fence_proxy_async_smem();
  if (threadIdx.x < 32) tmem_alloc(&tbase_s, 512);
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    for (int i = 0; i < 4; ++i) mbar_init(&bar2[i], 1);
    mbar_fence_init();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tb = tbase_s;
  if (threadIdx.x == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(128, N, false);
    const uint32_t a = smem_u32(A), b = smem_u32(B);
    uint64_t ad[8], bd[8];
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      ad[kk] = sdesc_kmajor(a, kk);
      bd[kk] = sdesc_kmajor(b, kk);
    }
    if (MODE >= 1) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tb + 448 + kk * 8), "l"(ad[kk]));
    }
    long long t0 = clock64();
    for (int it = 0; it < ITER; ++it) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint32_t d = tb + (uint32_t)((kk % ND) * N);
        if (MODE == 0)
          umma_bf16_ss(d, ad[kk], bd[kk], idesc, 1);
        else if (MODE == 1)
          umma_ts(d, tb + 448 + kk * 8, bd[kk], idesc, 1);
      }
      if (MODE == 2) umma_ts8(tb, tb + 448, bd, idesc);
      if (CM >= 1) umma_commit(&bar2[it & 3]);
      if (CM >= 2) umma_commit(&bar2[(it + 1) & 3]);
      if (CM >= 3) {  // wait for the commit of 2 iterations ago (pipelined consumer pattern)
        if (it >= 2) mbar_wait(&bar2[(it - 2) & 3], ((it - 2) >> 2) & 1);
      }
    }
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
    stop = 1;
  }
  if (threadIdx.x >= 128 && threadIdx.x < 128 + 32 * LDW) {
    // loader warps: continuous 32x32b.x32 TMEM loads from columns 256.. (lane quarter = warp % 4)
    const int w = threadIdx.x / 32;
    const uint32_t ta = tb + ((uint32_t)((w & 3) * 32) << 16) + 256 + (w >> 2) * 32;
    uint32_t r[32];
    float acc = 0.f;
    while (!stop) {
      tmem_ld32(ta, r);
      tmem_wait_ld();
      acc += __uint_as_float(r[0]) + __uint_as_float(r[31]);
    }
    if (acc == 12345.f) out[0] = 0;
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x < 32) tmem_dealloc(tb, 512);
}

template <int MODE, int N, int ND, int LDW = 0, int CM = 0>
void run(const char* name, long long* d) {
  cudaFuncSetAttribute(kern<MODE, N, ND, LDW, CM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  kern<MODE, N, ND, LDW, CM><<<148, 384, 96 * 1024>>>(d);
  kern<MODE, N, ND, LDW, CM><<<148, 384, 96 * 1024>>>(d);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
  double s = 0;
  for (int i = 0; i < 148; ++i) s += h[i];
  s /= 148;
  printf("%-22s %7.1f cyc/MMA (ideal %5.1f)  %s\n", name, s / (ITER * 8), 128.0 * N / 256.0,
         cudaGetErrorString(e));
}

int main() {
  long long* d;
  cudaMalloc(&d, 148 * 8);
  run<0, 128, 1>("SS N=128", d);
  run<0, 64, 1>("SS N=64", d);
  run<0, 256, 1>("SS N=256", d);
  run<1, 128, 1>("TS N=128", d);
  run<1, 128, 2>("TS N=128 2 acc", d);
  run<1, 64, 1>("TS N=64", d);
  run<1, 64, 2>("TS N=64 2 acc", d);
  run<1, 256, 1>("TS N=256", d);
  run<1, 128, 1, 4>("TS N=128 + 4 ld warps", d);
  run<1, 128, 1, 8>("TS N=128 + 8 ld warps", d);
  run<0, 128, 1, 8>("SS N=128 + 8 ld warps", d);
  run<1, 64, 1, 8>("TS N=64 + 8 ld warps", d);
  run<1, 128, 1, 0, 1>("TS N=128 commit/8", d);
  run<1, 128, 1, 0, 2>("TS N=128 2 commits/8", d);
  run<1, 64, 1, 0, 2>("TS N=64 2 commits/8", d);
  return 0;
}
