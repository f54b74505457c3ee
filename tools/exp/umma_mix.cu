// Microbenchmark: the verify kernel's MMA mix (per tile: 8 x QK M128 N64 TS
// K-major into S, 8 x PV M128 N128 TS MN-major into O) issued (a) by one
// thread, (b) by two threads (QK / PV issuers), (c) as (b) with 8 warps doing
// tcgen05.ld/st traffic on other TMEM columns, (d) as (b) with the 8 warps
// hammering shared memory.  clock64 per tile.
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
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t I, int acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
               ::"r"(d), "r"(a), "l"(b), "r"(I), "r"(acc));
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t I, int acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
               ::"r"(d), "l"(a), "l"(b), "r"(I), "r"(acc));
}
__device__ volatile int g_stop;

template <int MODE, int SS>
__global__ void __launch_bounds__(384, 1) k(long long* out, int tiles) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar[3];
  __shared__ volatile int done;
  const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
  for (int i = threadIdx.x; i < 160 * 1024 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
  const uint32_t b0 = (uint32_t)__cvta_generic_to_shared(&bar[0]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0 + 8));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0 + 16));
    done = 0;
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tm = tslot;
  constexpr uint32_t IQK = idesc_bf16(128, 64, 0), IPV = idesc_bf16(128, 128, 1);
  auto qk = [&](int t) {
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t bd = sdesc(sb + 32768 + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024);
      if (SS) mma_ss(tm + (t & 1) * 64, sdesc(sb + (kk >> 2) * 16384 + (kk & 3) * 32, 16, 1024), bd, IQK, kk > 0);
      else mma_ts(tm + (t & 1) * 64, tm + 256 + kk * 8, bd, IQK, kk > 0);
    }
  };
  auto pv = [&](int t) {
    for (int kk = 0; kk < 8; ++kk) {
      const uint64_t bd = sdesc(sb + 65536 + (kk & 3) * 2048, 8192, 1024);
      if (SS) mma_ss(tm + 128, sdesc(sb + 98304 + (kk >> 2) * 8192 + (kk & 3) * 32, 16, 1024), bd, IPV, 1);
      else mma_ts(tm + 128, tm + 320 + (t & 1) * 64 + kk * 8, bd, IPV, 1);
    }
  };
  long long t0 = clock64();
  if (MODE == 0) {
    if (threadIdx.x == 0) {
      for (int t = 0; t < tiles; ++t) { qk(t); pv(t); }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b0));
    }
  } else {
    if (threadIdx.x == 32) {
      for (int t = 0; t < tiles; ++t) qk(t);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b0));
    } else if (threadIdx.x == 352) {
      for (int t = 0; t < tiles; ++t) pv(t);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(b0 + 8));
    } else if (warp >= 2 && warp <= 9 && MODE >= 2) {
      // background traffic until the issuers finish
      const uint32_t la = (uint32_t)((warp & 3) * 32) << 16;
      float acc = 0.f;
      while (done < 2) {
        if (MODE == 2) {
          uint32_t r[32];
          asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
              : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31])
              : "r"(tm + la + 448 + (warp >= 6 ? 32 : 0)));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          for (int j = 0; j < 32; ++j) acc += __uint_as_float(r[j]);
        } else if (MODE == 4) {
          uint32_t ok;
          asm volatile("{\n\t.reg .pred P1;\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0;\n\tselp.u32 %0, 1, 0, P1;\n}" : "=r"(ok) : "r"(b0 + 16));
          acc += ok;
        } else if (MODE == 5) {
          asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};"
              :: "r"(tm + la + 448 + (warp >= 6 ? 32 : 0)), "r"(lane));
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        } else {
          const float* s = (const float*)(smem + 131072);
          for (int j = 0; j < 32; ++j) acc += s[(lane + j * 32 + warp * 7) & 4095];
        }
      }
      if (acc == 1234.5f) out[5] = 1;
    }
    if (threadIdx.x == 32 || threadIdx.x == 352) {
      asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n}" ::"r"(b0 + (threadIdx.x == 32 ? 0 : 8)));
      atomicAdd((int*)&done, 1);
    }
  }
  if (threadIdx.x == 0 && MODE == 0)
    asm volatile("{\n\t.reg .pred P1;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n}" ::"r"(b0));
  if ((threadIdx.x == 0 && MODE == 0) || threadIdx.x == 32 || threadIdx.x == 352) {
    long long t1 = clock64();
    if (blockIdx.x == 0) out[threadIdx.x == 352 ? 1 : 0] = t1 - t0;
  }
  __syncthreads();   // warps 2-9 spin on done until issuers arrive? no: set done first
  if (warp == 1) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

// done must be set before the final __syncthreads: use a second kernel layout
template <int MODE, int SS>
void run(const char* name) {
  long long* d; cudaMalloc(&d, 64); cudaMemset(d, 0, 64);
  auto f = k<MODE, SS>;
  cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
  const int tiles = 512;
  f<<<148, 384, 160 * 1024>>>(d, tiles);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%-36s %s: %.0f / %.0f cyc per tile (ideal 8*55.5+8*64 = 956) %s\n", name, SS ? "SS" : "TS",
         (double)h[0] / tiles, (double)h[1] / tiles, cudaGetErrorString(e));
  cudaFree(d);
}
int main() {
  run<0, 0>("one issuer");
  run<0, 1>("one issuer");
  run<1, 0>("two issuers");
  run<1, 1>("two issuers");
  run<2, 0>("two issuers + tcgen05.ld traffic");
  run<2, 1>("two issuers + tcgen05.ld traffic");
  run<3, 0>("two issuers + smem traffic");
  run<3, 1>("two issuers + smem traffic");
  run<4, 0>("two issuers + mbarrier spin");
  run<5, 0>("two issuers + tcgen05.st traffic");
  return 0;
}
