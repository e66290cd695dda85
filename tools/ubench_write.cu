// Write-bandwidth microbenchmark on B200: plain 16-byte stores, streaming
// (.cs) stores and TMA bulk stores (smem -> global), 256 MB buffers.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_write tools/ubench_write.cu
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__global__ void st_plain(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint4(1, 2, 3, (uint32_t)i);
}
__global__ void st_cs(uint4* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    __stcs(p + i, make_uint4(1, 2, 3, (uint32_t)i));
}
__global__ void st_8b(uint2* p, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    p[i] = make_uint2(1, (uint32_t)i);
}
__global__ void st_tma(char* p, size_t bytes) {
  extern __shared__ __align__(128) char buf[];
  const int chunk = 32768;
  for (int i = threadIdx.x; i < chunk / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(buf)[i] = i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    for (size_t off = (size_t)blockIdx.x * chunk; off < bytes; off += (size_t)gridDim.x * chunk) {
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + off),
                   "r"((uint32_t)__cvta_generic_to_shared(buf)), "r"(chunk) : "memory");
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  }
}
__global__ void rd_wr(const uint4* a, uint4* b, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    b[i] = a[i];
}

int main(int argc, char** argv) {
  const size_t bytes = (argc > 1 ? (size_t)atoll(argv[1]) : 256ull) << 20;  // MiB
  printf("buffer %zu MiB\n", bytes >> 20);
  char *a, *b;
  cudaMalloc(&a, bytes);
  cudaMalloc(&b, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](const char* name, auto fn, double moved) {
    for (int i = 0; i < 3; ++i) fn();
    cudaEventRecord(e0);
    for (int i = 0; i < 20; ++i) fn();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s %8.1f GB/s\n", name, moved * 20 / (ms * 1e-3) / 1e9);
  };
  const size_t n16 = bytes / 16;
  for (int bpsm : {4, 8, 16}) {
    char nm[64];
    snprintf(nm, 64, "st.128 plain  %d CTA/SM", bpsm);
    run(nm, [&] { st_plain<<<148 * bpsm, 256>>>((uint4*)a, n16); }, bytes);
    snprintf(nm, 64, "st.128 .cs    %d CTA/SM", bpsm);
    run(nm, [&] { st_cs<<<148 * bpsm, 256>>>((uint4*)a, n16); }, bytes);
    snprintf(nm, 64, "st.64 plain   %d CTA/SM", bpsm);
    run(nm, [&] { st_8b<<<148 * bpsm, 256>>>((uint2*)a, bytes / 8); }, bytes);
  }
  cudaFuncSetAttribute(st_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
  run("tma bulk store 32KB", [&] { st_tma<<<148 * 4, 128, 32768>>>(a, bytes); }, bytes);
  run("copy (read+write bytes)", [&] { rd_wr<<<148 * 8, 256>>>((uint4*)a, (uint4*)b, n16); }, 2.0 * bytes);
  return 0;
}
