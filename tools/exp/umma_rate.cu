// Microbenchmark: tcgen05.mma kind::f16 issue rate for the shapes the verify
// kernel uses (M=128; N=64/128/256; A from smem (SS) or TMEM (TS); B K-major or
// MN-major, SWIZZLE_128B).  One CTA per SM, clock64 around n MMAs + commit.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int b_mn_major) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn_major << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, int TS, int BMN>
__global__ void __launch_bounds__(128, 1) k(long long* out, int n) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
  const uint32_t barp = (uint32_t)__cvta_generic_to_shared(&bar);
  if (threadIdx.x == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(barp));
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  if (threadIdx.x == 0) {
    constexpr uint32_t I = idesc_bf16(128, N, BMN);
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
      const uint64_t bd = BMN ? sdesc(sb + 32768 + (i & 3) * 2048, 8192, 1024)
                              : sdesc(sb + 32768 + (i & 3) * 32, 16, 1024);
      if (TS) {
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(tm), "r"(tm + 256 + (i & 7) * 8), "l"(bd), "r"(I), "r"(i > 0 ? 1 : 0));
      } else {
        const uint64_t ad = sdesc(sb + (i & 3) * 32, 16, 1024);
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                     "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(tm), "l"(ad), "l"(bd), "r"(I), "r"(i > 0 ? 1 : 0));
      }
    }
    long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(barp));
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n}" ::"r"(barp));
    long long t2 = clock64();
    if (blockIdx.x == 0) { out[0] = t1 - t0; out[1] = t2 - t0; }
  }
  __syncthreads();
  if (threadIdx.x < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int TS, int BMN>
void run(const char* name, int grid) {
  long long* d; cudaMalloc(&d, 16);
  auto f = k<N, TS, BMN>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int n = 4096;
  f<<<grid, 128, 96 * 1024>>>(d, n);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  f<<<grid, 128, 96 * 1024>>>(d, n);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  double macs = 128.0 * N * 16 * n;
  printf("%-26s grid %3d: issue %6.1f cyc/mma, done %6.1f cyc/mma, %.0f MAC/cyc/SM, %.1f TFLOP/s chip (%s)\n",
         name, grid, (double)h[0] / n, (double)h[1] / n, macs / h[1],
         2 * macs * grid / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  for (int g : {1, 148}) {
    run<64, 0, 0>("SS N=64 B K-major", g);
    run<64, 1, 0>("TS N=64 B K-major", g);
    run<128, 0, 0>("SS N=128 B K-major", g);
    run<128, 1, 0>("TS N=128 B K-major", g);
    run<128, 0, 1>("SS N=128 B MN-major", g);
    run<128, 1, 1>("TS N=128 B MN-major", g);
    run<256, 0, 0>("SS N=256 B K-major", g);
    run<256, 1, 0>("TS N=256 B K-major", g);
  }
  return 0;
}
