// SPDX-License-Identifier: Apache-2.0
// Microbenchmark: per-SM throughput of MUFU.EX2 (ex2.approx.ftz.f32), of the FMA-pipe
// polynomial 2^x (ex2_poly of fine_fwd_sm100.cu) and of FFMA2, on one SM-resident CTA
// per SM with 8..32 warps. Answers whether the d = 64 softmax work (8192 exp2 per pair of
// 64x64 tiles) is bound by the MUFU pipe on B200.
#include <cstdint>
#include <cstdio>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// ex2.approx.f16x2: two exponentials per MUFU instruction (half precision)
__device__ __forceinline__ float ex2h2(float x) {
  const __half2 h = __floats2half2_rn(x, x * 0.5f);
  uint32_t r;
  asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(r) : "r"(*reinterpret_cast<const uint32_t*>(&h)));
  const __half2 o = *reinterpret_cast<const __half2*>(&r);
  return __low2float(o) + __high2float(o);
}
__device__ __forceinline__ float ex2_poly(float x) {
  x = fmaxf(x, -120.f);
  const float t = x + 12582912.f;
  const float f = x - (t - 12582912.f);
  const float p = fmaf(fmaf(fmaf(0.05508872f, f, 0.24260436f), f, 0.6932763f), f, 0.99992895f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

template <int MODE>
__global__ void bench(float* out, long long* cycles, int iters) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = -0.001f * (threadIdx.x + i);
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (MODE == 0) a[i] = ex2(a[i]) - 1.0f;
      if (MODE == 1) a[i] = ex2_poly(a[i]) - 1.0f;
      if (MODE == 2) a[i] = fmaf(a[i], 0.999f, -0.0001f);
      if (MODE == 3) a[i] = ex2h2(a[i]) - 2.0f;
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE>
void run(const char* name, int warps) {
  const int sms = 148, iters = 4096, thr = warps * 32;
  float* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(float) * sms * thr);
  cudaMalloc(&cyc, sizeof(long long) * sms);
  bench<MODE><<<sms, thr>>>(out, cyc, 16);
  bench<MODE><<<sms, thr>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h[148];
  cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
  double avg = 0;
  for (int i = 0; i < sms; ++i) avg += double(h[i]) / sms;
  const double ops = double(iters) * 8 * thr * (MODE == 3 ? 2 : 1);
  printf("%-10s warps=%2d: %.2f results/cycle/SM (%.0f cycles)\n", name, warps, ops / avg, avg);
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {8, 16, 32}) {
    run<0>("mufu.ex2", w);
    run<1>("poly_ex2", w);
    run<2>("ffma", w);
    run<3>("ex2.f16x2", w);
  }
  return 0;
}
