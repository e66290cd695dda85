// Shared device helpers for the HQMQ sm_100a kernels.
//
// Exactness rules (SURVEY.md §8a "exact arithmetic contract"): every fp64
// operation that must match the reference's numpy arithmetic goes through
// the explicit round-to-nearest intrinsics (__dmul_rn / __dadd_rn /
// __ddiv_rn / __dsqrt_rn) so nvcc can never contract it into an FMA.
#pragma once

#include <utility>

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/hqmq_b200.h"

namespace hqmq {

constexpr int kGroupOrder = 24;  // |2T|, hurwitz.py:25
constexpr int kWarp = 32;

// ---------------------------------------------------------------- input
template <typename T>
struct In;
template <>
struct In<__half> {
  static __device__ __forceinline__ double d(__half v) { return (double)__half2float(v); }
  static __device__ __forceinline__ float f(__half v) { return __half2float(v); }
};
template <>
struct In<__nv_bfloat16> {
  static __device__ __forceinline__ double d(__nv_bfloat16 v) { return (double)__bfloat162float(v); }
  static __device__ __forceinline__ float f(__nv_bfloat16 v) { return __bfloat162float(v); }
};
template <>
struct In<float> {
  static __device__ __forceinline__ double d(float v) { return (double)v; }
  static __device__ __forceinline__ float f(float v) { return v; }
};
template <>
struct In<double> {
  static __device__ __forceinline__ double d(double v) { return v; }
  static __device__ __forceinline__ float f(double v) { return (float)v; }
};

// Load the 4 elements of chunk c of a token row (zero padding past head_dim,
// codec.py:197-205).  `row` points at the first element of the token.
template <typename T>
__device__ __forceinline__ void load_chunk(const T* __restrict__ row, int c, int head_dim,
                                           bool aligned4, T (&v)[4]) {
  const int e0 = 4 * c;
  if (aligned4) {
    if constexpr (sizeof(T) == 2) {
      uint2 raw = __ldg(reinterpret_cast<const uint2*>(row + e0));
      const T* p = reinterpret_cast<const T*>(&raw);
      v[0] = p[0]; v[1] = p[1]; v[2] = p[2]; v[3] = p[3];
    } else if constexpr (sizeof(T) == 4) {
      float4 raw = __ldg(reinterpret_cast<const float4*>(row + e0));
      const T* p = reinterpret_cast<const T*>(&raw);
      v[0] = p[0]; v[1] = p[1]; v[2] = p[2]; v[3] = p[3];
    } else {
      double2 a = __ldg(reinterpret_cast<const double2*>(row + e0));
      double2 b = __ldg(reinterpret_cast<const double2*>(row + e0 + 2));
      v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    }
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = e0 + i;
      v[i] = e < head_dim ? row[e] : T(0.0f);
    }
  }
}

// r = sqrt(((x0*x0 + x1*x1) + x2*x2) + x3*x3), numpy's left-to-right 4-term
// reduce (codec.py:252), no FMA.
__device__ __forceinline__ double exact_norm(const double (&x)[4]) {
  double s = __dmul_rn(x[0], x[0]);
  s = __dadd_rn(s, __dmul_rn(x[1], x[1]));
  s = __dadd_rn(s, __dmul_rn(x[2], x[2]));
  s = __dadd_rn(s, __dmul_rn(x[3], x[3]));
  return __dsqrt_rn(s);
}

// ((u0*c0 + u1*c1) + u2*c2) + u3*c3 in fp64, no FMA (_kernels.pyx:35-40).
__device__ __forceinline__ double exact_dot(const double (&u)[4], const double* c) {
  double s = __dmul_rn(u[0], c[0]);
  s = __dadd_rn(s, __dmul_rn(u[1], c[1]));
  s = __dadd_rn(s, __dmul_rn(u[2], c[2]));
  s = __dadd_rn(s, __dmul_rn(u[3], c[3]));
  return s;
}

// Radius quantum (radius.py:35-47): clip(floor((r*top)/sigma_w + 0.5), 0, top).
__device__ __forceinline__ uint32_t exact_quantum(double r, double sigma_w, double top) {
  double v = __dadd_rn(__ddiv_rn(__dmul_rn(r, top), sigma_w), 0.5);
  double q = floor(v);
  q = q < 0.0 ? 0.0 : (q > top ? top : q);
  return (uint32_t)q;
}

// ------------------------------------------------------------- bit streams
// Read `width` (1..32) bits at absolute bit offset `bit` of an LSB-first
// stream stored as little-endian 32-bit words (kvpack.py:66-76).  Streams are
// allocated with one padding word so the second load is always in bounds.
__device__ __forceinline__ uint32_t read_bits(const uint32_t* __restrict__ words, uint64_t bit,
                                              int width) {
  const uint64_t w = bit >> 5;
  const uint32_t sh = (uint32_t)(bit & 31);
  const uint32_t lo = __ldg(words + w);
  const uint32_t hi = __ldg(words + w + 1);
  const uint32_t v = __funnelshift_r(lo, hi, sh);
  return width == 32 ? v : (v & ((1u << width) - 1u));
}

// --------------------------------------------------------------- reductions
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Argmax with the reference's tie-break: larger score wins, equal scores go to
// the lower flat index (strict '>' in ascending order, _kernels.pyx:41).
__device__ __forceinline__ void warp_argmax_lowest(double& score, long long& idx) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double s2 = __shfl_xor_sync(0xffffffffu, score, o);
    long long i2 = __shfl_xor_sync(0xffffffffu, idx, o);
    if (s2 > score || (s2 == score && i2 < idx)) {
      score = s2;
      idx = i2;
    }
  }
}

// ------------------------------------------------ TMA bulk copy / mbarrier
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
// 1-D bulk copy global -> shared (TMA, UBLKCP), completion counted on `bar`.
// dst/src 16-byte aligned, bytes a multiple of 16.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Ring-stage release count: acq_rel, so a warp's reads of the stage happen
// before the last releaser's refill (which then fences into the async proxy).
__device__ __forceinline__ uint32_t stage_release(unsigned int* count) {
  uint32_t old;
  asm volatile("atom.acq_rel.cta.shared::cta.add.u32 %0, [%1], 1;" : "=r"(old) : "r"(smem_u32(count)) : "memory");
  return old;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase), "r"(0x989680u)
      : "memory");
}

// Programmatic dependent launch (PDL): a kernel launched with launch_pdl may
// start while the previous kernel of its stream drains; it sets itself up
// (barriers, constant tables) and then calls pdl_wait() before it touches
// anything an earlier kernel produced.  pdl_trigger() lets the next
// PDL-launched kernel of the stream start its own set-up early.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
#ifdef HQMQ_NO_PDL  // diagnostic builds: plain stream order
  cfg.numAttrs = 0;
#else
  cfg.numAttrs = 1;
#endif
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Records the CUDA error text for hqmq_last_error() and returns HQMQ_ERR_CUDA.
int record_cuda_error(cudaError_t e);
inline int check_launch() {
  const cudaError_t e = cudaGetLastError();
  return e == cudaSuccess ? HQMQ_OK : record_cuda_error(e);
}

__host__ __device__ __forceinline__ int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

}  // namespace hqmq
