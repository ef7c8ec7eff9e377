// Microbenchmark: which pipe does the fp32 -> bf16x2 pack (F2FP) use on sm_100a?
// Each kernel runs ITER iterations over 8 independent chains per thread, 256
// threads per CTA, one CTA per SM; reports cycles per warp-instruction per SMSP.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

constexpr int ITER = 4096;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack(float a, float b) {
  uint32_t r;
  asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(b), "f"(a));
  return r;
}
__device__ __forceinline__ uint32_t pack_int(float a, float b) {
  // RNE by integer arithmetic (finite inputs): t = x + 0x7fff + lsb(x >> 16)
  uint32_t ua = __float_as_uint(a), ub = __float_as_uint(b);
  ua += 0x7fffu + ((ua >> 16) & 1u);
  ub += 0x7fffu + ((ub >> 16) & 1u);
  return __byte_perm(ua, ub, 0x7632);
}

__device__ __forceinline__ uint32_t ex2h2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}
__device__ __forceinline__ uint32_t ex2bf2(uint32_t x) {
  uint32_t y;
  asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(x));
  return y;
}

template <int MODE>
__global__ void kern(float* out, long long* cyc) {
  float x[8];
  uint32_t acc = 0;
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3f + i * 1e-4f;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < ITER; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) x[i] = ex2(x[i]) * -0.5f;
      if (MODE == 1) {
        acc ^= pack(x[i], x[(i + 1) & 7]);
        x[i] = __uint_as_float(__float_as_uint(x[i]) ^ (acc & 1u));
      }
      if (MODE == 2) {  // softmax mix: 2 ex2 per pack
        x[i] = ex2(x[i]) * -0.5f;
        if (i & 1) acc ^= pack(x[i - 1], x[i]);
      }
      if (MODE == 3) {  // softmax mix with integer pack
        x[i] = ex2(x[i]) * -0.5f;
        if (i & 1) acc ^= pack_int(x[i - 1], x[i]);
      }
      if (MODE == 5) x[i] = __uint_as_float(ex2h2(__float_as_uint(x[i])) ^ 0x80008000u);
      if (MODE == 6) x[i] = __uint_as_float(ex2bf2(__float_as_uint(x[i])) ^ 0x80008000u);
      if (MODE == 4) {
        acc ^= pack_int(x[i], x[(i + 1) & 7]);
        x[i] = __uint_as_float(__float_as_uint(x[i]) ^ (acc & 1u));
      }
    }
  }
  long long t1 = clock64();
  __syncthreads();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += x[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, double ops_per_iter_thread) {
  float* out;
  long long* cyc;
  cudaMalloc(&out, 148 * 256 * 4);
  cudaMalloc(&cyc, 148 * 8);
  kern<MODE><<<148, 256>>>(out, cyc);
  kern<MODE><<<148, 256>>>(out, cyc);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  double c = 0;
  for (int i = 0; i < 148; ++i) c += h[i];
  c /= 148;
  // 8 warps per SM -> 2 warps per SMSP
  double warp_instr_per_smsp = 2.0 * ITER * ops_per_iter_thread;
  printf("%-28s cycles %.0f  cycles per warp-op per SMSP %.2f  lane-ops/clk/SM %.1f\n", name, c,
         c / warp_instr_per_smsp, 256.0 * ITER * ops_per_iter_thread / c);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  run<0>("ex2 (MUFU)", 8);
  run<1>("cvt.rn.bf16x2 pack", 8);
  run<4>("integer RNE pack", 8);
  run<2>("2 ex2 + 1 cvt pack (per pair)", 8);
  run<3>("2 ex2 + 1 int pack (per pair)", 8);
  run<5>("ex2.approx.f16x2 (2 results)", 8);
  run<6>("ex2.approx.ftz.bf16x2 (2 results)", 8);
  return 0;
}
