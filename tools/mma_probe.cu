// mma_probe.cu -- how long does one tcgen05.mma (kind::tf32 K = 8, kind::f16 K = 16; operands K-major, no swizzle) take as a
// function of its M and N? One CTA per SM, one thread issues `chain` MMAs into the same accumulator, commits, waits.
// Operand contents are irrelevant (uninitialised shared memory is fine: only the issue rate is read).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mma_probe tools/mma_probe.cu && /tmp/mma_probe
// Measurement helper, not product code.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <utility>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t make_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ uint32_t make_idesc(int m, int n, int f16) {  // D = F32; A, B = TF32 (2) or F16 (0)
  const uint32_t ab = f16 ? 0u : 2u;
  return (1u << 4) | (ab << 7) | (ab << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void mma_tf32(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ bool mbar_wait(uint64_t* bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  for (int spin = 0; spin < (1 << 24); ++spin) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                 : "=r"(ok)
                 : "r"(addr), "r"(parity)
                 : "memory");
    if (ok) return true;
  }
  return false;
}

// accs = number of distinct accumulators the chain rotates over (1 = every MMA depends on the previous one's D)
// tmem_cols: 512 with one CTA per SM, 256 with two (both then issue into the SM's one tensor pipe)
__global__ void __launch_bounds__(128, 2) probe(long long* out, int m, int n, int chain, int accs, int reps, int f16, uint32_t tmem_cols) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x;
  for (int i = tid; i < 48 * 1024 / 4; i += 128) reinterpret_cast<float*>(smem)[i] = 1.0f / (float)(1 + (i & 255));
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1u) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&slot)), "r"(tmem_cols) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = slot;
  long long best = 1ll << 60;
  bool ok = true;
  if (tid == 0) {
    // A: m rows, B: n rows, both [8-row group][K core 2][8 rows x 16 B]: SBO = 256, LBO = 128
    const uint32_t a_addr = smem_u32(smem), b_addr = a_addr + 16 * 1024;
    const uint64_t da = make_desc(a_addr, 128, 256), db = make_desc(b_addr, 128, 256);
    const uint32_t idesc = make_idesc(m, n, f16);
    for (int r = 0; r < reps && ok; ++r) {
      const long long t0 = clock64();
      if (f16)
        for (int i = 0; i < chain; ++i) mma_f16(tm + (uint32_t)((i % accs) * n), da, db, idesc, i >= accs ? 1u : 0u);
      else
        for (int i = 0; i < chain; ++i) mma_tf32(tm + (uint32_t)((i % accs) * n), da, db, idesc, i >= accs ? 1u : 0u);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
      ok = mbar_wait(&bar, (uint32_t)(r & 1));
      const long long t1 = clock64();
      if (t1 - t0 < best) best = t1 - t0;
    }
    if (blockIdx.x == 0) out[0] = ok ? best : -1;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(tmem_cols) : "memory");
  }
}

int main() {
  long long* d;
  cudaMalloc(&d, 8);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
  const int shapes[][2] = {{128, 16}, {128, 32}, {128, 48}, {128, 64}, {128, 96}, {128, 128}, {128, 176}, {128, 256},
                           {64, 16},  {64, 32},  {64, 64},  {64, 128}, {64, 192}, {64, 256}};
  printf("tcgen05.mma, cycles per MMA (chain of 64 minus chain of 32, over 32), one CTA per SM\n");
  for (int f16 : {0, 1})
  for (auto& s : shapes) {
    for (int accs : {1}) {
      if (accs * s[1] > 512) continue;
      long long c[2] = {0, 0};
      int k = 0;
      for (int chain : {32, 64}) {
        probe<<<148, 128, 48 * 1024>>>(d, s[0], s[1], chain, accs, 20, f16, 512u);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("M=%d N=%d: %s\n", s[0], s[1], cudaGetErrorString(e));
          return 1;
        }
        cudaMemcpy(&c[k++], d, 8, cudaMemcpyDeviceToHost);
      }
      const double per = (double)(c[1] - c[0]) / 32.0;
      printf("%s M=%3d N=%3d accumulators=%d: %7.1f cycles/MMA  (%.0f MAC/clk; chain32 %lld, chain64 %lld)\n", f16 ? "f16 K=16 " : "tf32 K=8 ", s[0], s[1], accs, per,
             (double)s[0] * s[1] * (f16 ? 16 : 8) / per, c[0], c[1]);
    }
  }
  // two CTAs per SM, each with its own issuing thread: is the 150 cycles a per-thread issue cost or the pipe's?
  for (auto& s : {std::pair<int, int>{128, 32}, {128, 176}, {64, 48}}) {
    long long c[2] = {0, 0};
    int k = 0;
    for (int chain : {32, 64}) {
      probe<<<296, 128, 48 * 1024>>>(d, s.first, s.second, chain, 1, 20, 0, 256u);
      if (cudaDeviceSynchronize() != cudaSuccess) return 1;
      cudaMemcpy(&c[k++], d, 8, cudaMemcpyDeviceToHost);
    }
    printf("tf32 K=8  M=%3d N=%3d, TWO CTAs per SM issuing at once: %7.1f cycles/MMA per CTA\n", s.first, s.second,
           (double)(c[1] - c[0]) / 32.0);
  }
  return 0;
}
