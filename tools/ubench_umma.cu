// Standalone check of the hand-written tcgen05 path used by the encode search:
// D[128 x 256] (fp32, TMEM) = A[128 x 16] . B[256 x 16]^T (fp16, K-major,
// SWIZZLE_NONE canonical layout), one CTA, one elected thread issues the MMA.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_umma tools/ubench_umma.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <math.h>

#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
// K-major, no swizzle: element (r, k) at (r/8)*SBO + (k/8)*LBO + (r%8)*16 + (k%8)*2
constexpr uint32_t kLBO = 128, kSBO = 256;
__device__ __forceinline__ uint32_t kmaj_off(int r, int k) {
  return (r >> 3) * kSBO + (k >> 3) * kLBO + (r & 7) * 16 + (k & 7) * 2;
}
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_u32(p) >> 4) & 0x3FFF);
  d |= (uint64_t)((kLBO >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((kSBO >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  return d;                // base offset 0, lbo mode 0, layout SWIZZLE_NONE
}
__host__ __device__ constexpr uint32_t instr_desc(int M, int N) {
  return (1u << 4)                     // D = F32
         | (0u << 7) | (0u << 10)      // A, B = F16
         | ((uint32_t)(N >> 3) << 17)  // N
         | ((uint32_t)(M >> 4) << 24); // M
}

__global__ void umma_test(const __half* A, const __half* B, float* D) {
  __shared__ __align__(1024) unsigned char sa[128 * 32];
  __shared__ __align__(1024) unsigned char sb[256 * 32];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int i = tid; i < 128 * 16; i += blockDim.x) {
    const int r = i / 16, k = i % 16;
    *reinterpret_cast<__half*>(sa + kmaj_off(r, k)) = A[i];
  }
  for (int i = tid; i < 256 * 16; i += blockDim.x) {
    const int r = i / 16, k = i % 16;
    *reinterpret_cast<__half*>(sb + kmaj_off(r, k)) = B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint64_t da = smem_desc(sa), db = smem_desc(sb);
    const uint32_t idesc = instr_desc(128, 256);
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
        "l"(da), "l"(db), "r"(idesc), "r"(0));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&bar)));
  }
  asm volatile(
      "{\n\t.reg .pred P1;\n\tW:\n\tmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n\t"
      "@P1 bra D;\n\tbra W;\n\tD:\n\t}" ::"r"(smem_u32(&bar)));
  asm volatile("tcgen05.fence::after_thread_sync;");
  for (int c0 = 0; c0 < 256; c0 += 32) {
    uint32_t v[32];
    const uint32_t addr = tmem + ((uint32_t)(warp * 32) << 16) + c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
          "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
          "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
          "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int j = 0; j < 32; ++j) D[(warp * 32 + (tid & 31)) * 256 + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256));
}

int main() {
  std::vector<__half> A(128 * 16), B(256 * 16);
  std::vector<float> Af(128 * 16), Bf(256 * 16), D(128 * 256);
  uint32_t st = 7;
  auto rnd = [&]() { st = st * 1664525u + 1013904223u; return (int)((st >> 20) % 7) - 3; };
  for (int i = 0; i < 128 * 16; ++i) { Af[i] = (float)rnd(); A[i] = __float2half(Af[i]); }
  for (int i = 0; i < 256 * 16; ++i) { Bf[i] = (float)rnd() * 0.5f; B[i] = __float2half(Bf[i]); }
  __half *dA, *dB;
  float* dD;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  umma_test<<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 256; ++n) {
      float ref = 0.f;
      for (int k = 0; k < 16; ++k) ref += Af[m * 16 + k] * Bf[n * 16 + k];
      if (ref != D[m * 256 + n] && bad++ < 5) printf("mismatch m=%d n=%d got %f want %f\n", m, n, D[m * 256 + n], ref);
    }
  printf("umma 128x256x16: %s (%d mismatches)\n", bad ? "FAIL" : "OK", bad);
  // accuracy of the split-fp16 rotation used by the encode search:
  // A row = [u1, u1, u2, 0], B row (column n) = [R1, R2, R1, 0] -> v ~= u.R
  double maxerr = 0.0;
  uint64_t s2 = 12345;
  auto uni = [&]() { s2 = s2 * 6364136223846793005ull + 1442695040888963407ull;
                     return ((s2 >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0; };
  for (int trial = 0; trial < 20; ++trial) {
    std::vector<double> u(128 * 4), R(4 * 256);
    for (int m = 0; m < 128; ++m) {
      double nn = 0; for (int i = 0; i < 4; ++i) { u[m * 4 + i] = uni(); nn += u[m * 4 + i] * u[m * 4 + i]; }
      nn = sqrt(nn); for (int i = 0; i < 4; ++i) u[m * 4 + i] = (float)(u[m * 4 + i] / nn);
    }
    for (int n = 0; n < 256; ++n) {
      double nn = 0; for (int i = 0; i < 4; ++i) { R[i * 256 + n] = uni(); nn += R[i * 256 + n] * R[i * 256 + n]; }
      nn = sqrt(nn); for (int i = 0; i < 4; ++i) R[i * 256 + n] = (float)(R[i * 256 + n] / nn);
    }
    for (int m = 0; m < 128; ++m)
      for (int i = 0; i < 4; ++i) {
        const __half h1 = __float2half((float)u[m * 4 + i]);
        const __half h2 = __float2half((float)u[m * 4 + i] - __half2float(h1));
        A[m * 16 + i] = h1; A[m * 16 + 4 + i] = h1; A[m * 16 + 8 + i] = h2; A[m * 16 + 12 + i] = __float2half(0.f);
      }
    for (int n = 0; n < 256; ++n)
      for (int i = 0; i < 4; ++i) {
        const float r = (float)R[i * 256 + n];
        const __half h1 = __float2half(r), h2 = __float2half(r - __half2float(h1));
        B[n * 16 + i] = h1; B[n * 16 + 4 + i] = h2; B[n * 16 + 8 + i] = h1; B[n * 16 + 12 + i] = __float2half(0.f);
      }
    cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
    umma_test<<<1, 128>>>(dA, dB, dD);
    cudaDeviceSynchronize();
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 256; ++n) {
        double ref = 0; for (int i = 0; i < 4; ++i) ref += u[m * 4 + i] * R[i * 256 + n];
        maxerr = fmax(maxerr, fabs(ref - (double)D[m * 256 + n]));
      }
  }
  printf("split-fp16 rotation max |err| vs fp64: %.3e\n", maxerr);
  return bad != 0;
}
