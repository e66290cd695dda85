// tcgen05.mma issue-rate microbenchmark (SS mode, fp16 -> fp32, M = 128,
// SWIZZLE_NONE canonical layouts with the strides the prefill kernel uses):
// one CTA per SM, one thread issues R x 8 back-to-back MMAs (K = 128 in
// 16-steps), cycles per instruction vs N.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_umma_tput tools/ubench_umma_tput.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(lbo >> 4) << 16) |
         ((uint64_t)(sbo >> 4) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t idesc(int M, int N, int bmn) {
  return (1u << 4) | ((uint32_t)bmn << 16) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, int BMN>
__global__ void tput(int reps, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = tid; i < (32768 + N * 256) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint32_t a = smem_u32(sm), b = a + 32768;
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t da = desc(a + kk * 256, 128, 2048);
        const uint64_t db = BMN ? desc(b + kk * 256, 128, 1024) : desc(b + kk * 256, 128, 2048);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tbase),
            "l"(da), "l"(db), "r"(idesc(128, N, BMN)), "r"(kk));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
            smem_u32(&bar)) : "memory");
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(256));
}

// TS mode: A (M = 128 x K = 16 fp16) from TMEM columns [256, 264 + 8 kk)
template <int N, int BMN>
__global__ void tput_ts(int reps, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = tid; i < (N * 256) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint32_t b = smem_u32(sm);
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const uint64_t db = BMN ? desc(b + kk * 256, 128, 1024) : desc(b + kk * 256, 128, 2048);
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tbase),
            "r"(tbase + 256 + kk * 8), "l"(db), "r"(idesc(128, N, BMN)), "r"(kk));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
            smem_u32(&bar)) : "memory");
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(512));
}

template <int N, int BMN>
void run_ts(const char* name) {
  const int reps = 2000, grid = 148;
  unsigned long long* d;
  cudaMalloc(&d, grid * 8);
  const int smem = N * 256;
  cudaFuncSetAttribute(tput_ts<N, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tput_ts<N, BMN><<<grid, 128, smem>>>(10, d);
  cudaDeviceSynchronize();
  tput_ts<N, BMN><<<grid, 128, smem>>>(reps, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("%-22s N=%3d: %6.1f cycles/MMA (floor %d) (%s)\n", name, N, (double)h[0] / (reps * 8.0), N / 2,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

// The prefill tile: 8 SS MMAs (S = Q K^T, N = 128, D -> TMEM buffer b) then 8
// TS MMAs (O += P V, A = P from TMEM buffer b', B MN-major) per iteration.
__global__ void tile_seq(int reps, unsigned long long* cyc) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  for (int i = tid; i < (3 * 32768) / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3c003c00u;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (tid == 0) {
    const uint32_t q = smem_u32(sm), k = q + 32768, v = q + 65536;
    const uint32_t tm = tbase;
    const unsigned long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
      const uint32_t sb = (uint32_t)(r % 3) * 128, pb = (uint32_t)((r + 1) % 3) * 128;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tm + sb),
            "l"(desc(q + kk * 256, 128, 2048)), "l"(desc(k + kk * 256, 128, 2048)), "r"(idesc(128, 128, 0)),
            "r"(kk));
#pragma unroll
      for (int kk = 0; kk < 8; ++kk)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + 384),
            "r"(tm + pb + kk * 8), "l"(desc(v + kk * 256, 128, 2048)), "r"(idesc(128, 128, 1)), "r"(1));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    asm volatile(
        "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
            smem_u32(&bar)) : "memory");
    cyc[blockIdx.x] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(512));
}

void run_tile() {
  const int reps = 1000, grid = 148;
  unsigned long long* d;
  cudaMalloc(&d, grid * 8);
  const int smem = 3 * 32768;
  cudaFuncSetAttribute(tile_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tile_seq<<<grid, 128, smem>>>(10, d);
  cudaDeviceSynchronize();
  tile_seq<<<grid, 128, smem>>>(reps, d);
  cudaDeviceSynchronize();
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  printf("prefill tile (8 SS N=128 + 8 TS N=128): %.0f cycles/tile (floor 1024) (%s)\n",
         (double)h[0] / reps, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

template <int N, int BMN>
void run(const char* name) {
  const int reps = 2000, grid = 148;
  unsigned long long* d;
  cudaMalloc(&d, grid * 8);
  const int smem = 32768 + N * 256;
  cudaFuncSetAttribute(tput<N, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  tput<N, BMN><<<grid, 128, smem>>>(10, d);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  tput<N, BMN><<<grid, 128, smem>>>(reps, d);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  unsigned long long h[148];
  cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
  const double per = (double)h[0] / (reps * 8.0);
  const double flops = 2.0 * 128 * N * 16 * reps * 8.0 * grid;
  printf("%-22s N=%3d: %6.1f cycles/MMA (floor %d), %7.1f TFLOP/s (%s)\n", name, N, per, N / 2,
         flops / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  run<64, 0>("SS K-major B");
  run<128, 0>("SS K-major B");
  run<256, 0>("SS K-major B");
  run<64, 1>("SS MN-major B");
  run<128, 1>("SS MN-major B");
  run<256, 1>("SS MN-major B");
  run_ts<64, 0>("TS K-major B");
  run_ts<128, 0>("TS K-major B");
  run_ts<128, 1>("TS MN-major B");
  run_ts<256, 1>("TS MN-major B");
  run_tile();
  return 0;
}
