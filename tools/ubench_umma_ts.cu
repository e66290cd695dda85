// Layout check for tcgen05.mma with the A operand in TMEM (kind::f16, M = 128,
// K = 16): A row m = TMEM lane m, 32-bit column c = fp16 pair (k = 2c, 2c+1).
// D[128 x 64] = A . B^T with B (64 x 16, K-major) in shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_umma_ts tools/ubench_umma_ts.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <math.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(lbo >> 4) << 16) |
         ((uint64_t)(sbo >> 4) << 32) | ((uint64_t)1 << 46);
}
constexpr int N = 64;

__global__ void ts_test(const __half* A, const __half* B, float* D, int acol_off) {
  __shared__ __align__(1024) unsigned char sb[N * 32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < N * 16; i += blockDim.x) {
    const int r = i / 16, k = i % 16;  // K-major, SBO 256 (2 k-groups per 8 rows), LBO 128
    *reinterpret_cast<__half*>(sb + (r >> 3) * 256 + (k >> 3) * 128 + (r & 7) * 16 + (k & 7) * 2) = B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "n"(128));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  // A row `tid` -> TMEM lane tid, columns [64 + acol_off, +8)
  uint32_t a[8];
  for (int c = 0; c < 8; ++c) {
    __half2 h = __halves2half2(A[tid * 16 + 2 * c], A[tid * 16 + 2 * c + 1]);
    a[c] = *reinterpret_cast<uint32_t*>(&h);
  }
  const uint32_t arow = tm + 64 + acol_off + ((uint32_t)(warp * 32) << 16);
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(arow),
               "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(a[4]), "r"(a[5]), "r"(a[6]), "r"(a[7]));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm),
        "r"(tm + 64 + acol_off), "l"(desc(smem_u32(sb), 128, 256)), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t@!P1 bra W;\n\t}" ::"r"(
          smem_u32(&bar)) : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t d[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]), "=r"(d[7])
                 : "r"(tm + c0 + ((uint32_t)(warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 8; ++j) D[tid * N + c0 + j] = __uint_as_float(d[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(128));
}

int main() {
  __half hA[128 * 16], hB[N * 16];
  for (int i = 0; i < 128 * 16; ++i) hA[i] = __float2half((float)((i * 37) % 17 - 8) / 8.f);
  for (int i = 0; i < N * 16; ++i) hB[i] = __float2half((float)((i * 11) % 13 - 6) / 4.f);
  __half *dA, *dB;
  float* dD;
  cudaMalloc(&dA, sizeof(hA));
  cudaMalloc(&dB, sizeof(hB));
  cudaMalloc(&dD, 128 * N * 4);
  cudaMemcpy(dA, hA, sizeof(hA), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB, sizeof(hB), cudaMemcpyHostToDevice);
  for (int off = 0; off <= 16; off += 16) {
    ts_test<<<1, 128>>>(dA, dB, dD, off);
    static float hD[128 * N];
    cudaError_t e = cudaMemcpy(hD, dD, sizeof(hD), cudaMemcpyDeviceToHost);
    double maxerr = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < 16; ++k) ref += (double)__half2float(hA[m * 16 + k]) * __half2float(hB[n * 16 + k]);
        maxerr = fmax(maxerr, fabs(ref - hD[m * N + n]));
      }
    printf("A in TMEM (col offset %d): max |err| = %g (%s)\n", off, maxerr, cudaGetErrorString(e));
  }
  return 0;
}
