#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a), rb = *reinterpret_cast<unsigned long long*>(&b),
                     rc = *reinterpret_cast<unsigned long long*>(&c), rd;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  return *reinterpret_cast<float2*>(&rd);
}
template <int MODE>
__global__ void k(float* out, int iters, float s) {
  float2 a[8];
  for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x + i, threadIdx.x - i);
  float2 b = make_float2(s, s * 0.5f);
  unsigned u[8];
  for (int i = 0; i < 8; ++i) u[i] = threadIdx.x * 7 + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (MODE == 0 || MODE == 2) { a[i].x = fmaf(a[i].x, b.x, b.y); a[i].y = fmaf(a[i].y, b.y, b.x); }
        else a[i] = ffma2(a[i], b, b);
        if (MODE == 2) { u[i] = __funnelshift_l(u[i], u[i], 3); }            // 1 ALU op per 2 FFMA
        if (MODE == 3) { u[i] = __funnelshift_l(u[i], u[i], 3); }            // 1 ALU op per FFMA2
        if (MODE == 4) { u[i] = __funnelshift_l(u[i], u[i], 3); u[(i + 1) & 7] = __funnelshift_l(u[(i + 1) & 7], u[(i + 1) & 7], 5); }  // 2 ALU per FFMA2
      }
  }
  long long t1 = clock64();
  float acc = 0;
  for (int i = 0; i < 8; ++i) acc += a[i].x + a[i].y + (float)u[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (float)(t1 - t0);
}
int main() {
  float* d; cudaMalloc(&d, 148 * 8 * 1024 * 4);
  for (int mode = 0; mode < 5; ++mode)
    for (int warps : {4, 8, 16, 32}) {
      cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
      int iters = 20000;
      auto launch = [&]() {
        switch (mode) {
          case 0: k<0><<<148, warps * 32>>>(d, iters, 1.0001f); break;
          case 1: k<1><<<148, warps * 32>>>(d, iters, 1.0001f); break;
          case 2: k<2><<<148, warps * 32>>>(d, iters, 1.0001f); break;
          case 3: k<3><<<148, warps * 32>>>(d, iters, 1.0001f); break;
          default: k<4><<<148, warps * 32>>>(d, iters, 1.0001f); break;
        }
      };
      launch(); cudaDeviceSynchronize();
      cudaEventRecord(e0); launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      float cyc; cudaMemcpy(&cyc, d, 4, cudaMemcpyDeviceToHost);
      double fma = 148.0 * warps * 32 * iters * 64 * 2;  // scalar FMAs
      printf("mode %s warps/SM %2d: %.3f ms, %.1f TFLOP/s, cycles %.0f, FMA/clk/SM %.1f\n", (const char*[]){"FFMA       ", "FFMA2      ", "FFMA+.5ALU ", "FFMA2+1ALU ", "FFMA2+2ALU "}[mode], warps, ms,
             fma * 2 / ms * 1e-9, cyc, warps * 32.0 * iters * 128 / cyc);
    }
  return 0;
}
