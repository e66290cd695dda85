// Shared pieces of the decode-attention kernels (attention.cu,
// attention_cluster.cu): parameter blocks, mma.sync helpers, fp16 radius
// codes and the shared-memory code-run reader.
#pragma once

#include <cstdint>

#include "common.cuh"

namespace hqmq {

struct AttView {
  const uint16_t* scales;
  const uint32_t* idxw;
  const uint32_t* radw;
  const uint32_t* flagw;
  const uint16_t* payloads;
  const uint32_t* tokoff;
  const float4* table;  // [Hkv][24S]
  const uint2* table16;  // optional fp16 copy [Hkv][24S]
  const double* table64;  // [Hkv][24S][4] fp64 (the fp64 path)
};

struct AttParams {
  int64_t B, Hq, Hkv, Tq, Tkv, D;
  int C, S, br, w, g, causal;
  float scale_log2;
  int splits;
  int64_t keys_per_split;
  int nrows;  // g * Tq
  const float* q;
  AttView k, v;
  float* out;
  float* part_o;   // [B*Hkv][rows][splits][D]
  float* part_ml;  // [B*Hkv][rows][splits][2]
  // paged cache (decode serving layout): per-sequence lengths and the block
  // table of 128-token pages per (sequence, kv head) row
  const int32_t* kv_lens;
  const int32_t* block_table;
  int max_pages;
  float o_scale;  // combine_kernel multiplies the merged O by this (1 unless a kernel defers a constant factor)
};

// D(16x8 fp32) += A(16x16 fp16, rows 8-15 zero) * B(16x8 fp16)
__device__ __forceinline__ void mma_rows8(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0,
                                          uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}
__device__ __forceinline__ void mma_full(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_half2(float lo, float hi) {
  const __half2 h = __floats2half2_rn(lo, hi);
  return *reinterpret_cast<const uint32_t*>(&h);
}
// (q, q) as fp16x2 for an integer radius code q < 1024, without the
// quarter-rate I2F: 0x6400 | q is the fp16 1024 + q (exact), minus 1024.
__device__ __forceinline__ uint32_t code_half2(uint32_t q) {
  const uint32_t biased = (q * 0x10001u) | 0x64006400u;
  const __half2 r = __hsub2(*reinterpret_cast<const __half2*>(&biased), __float2half2_rn(1024.f));
  return *reinterpret_cast<const uint32_t*>(&r);
}
__device__ __forceinline__ uint32_t hmul2u(uint32_t a, uint32_t b) {
  const __half2 r = __hmul2(*reinterpret_cast<const __half2*>(&a), *reinterpret_cast<const __half2*>(&b));
  return *reinterpret_cast<const uint32_t*>(&r);
}

// N codes of WIDTH bits starting at bit `bit` of a shared-memory stream
// (LSB-first 32-bit words): NW words are loaded, aligned by one runtime
// funnel shift, then every code sits at a compile-time position.
// The run starts at bit key*32*WIDTH + t*N*WIDTH (t < NT), so its in-word
// shift is (t*N*WIDTH) & 31 and the worst case is known at compile time.
__host__ __device__ constexpr int max_run_shift(int n, int width, int nt) {
  int m = 0;
  for (int t = 0; t < nt; ++t) m = ((t * n * width) & 31) > m ? ((t * n * width) & 31) : m;
  return m;
}
template <int N, int WIDTH, int NT>
struct CodeRun {
  static constexpr int kSpan = max_run_shift(N, WIDTH, NT) + N * WIDTH;  // bits to cover
  static constexpr int kNW = (kSpan + 31) / 32;                          // words loaded
  uint32_t r[kNW];
  __device__ __forceinline__ void load(const uint32_t* __restrict__ s, uint32_t bit) {
    const uint32_t* p = s + (bit >> 5);
    const uint32_t sh = bit & 31;
    uint32_t w[kNW + 1];
#pragma unroll
    for (int i = 0; i < kNW; ++i) w[i] = p[i];
    w[kNW] = 0u;
#pragma unroll
    for (int i = 0; i < kNW; ++i) r[i] = __funnelshift_r(w[i], w[i + 1], sh);
  }
  __device__ __forceinline__ uint32_t get(int i) const {
    const int b = i * WIDTH, wi = b >> 5, sh = b & 31;
    uint32_t v = sh == 0 ? r[wi] : __funnelshift_r(r[wi], wi + 1 < kNW ? r[wi + 1] : 0u, sh);
    return WIDTH == 32 ? v : (v & ((1u << WIDTH) - 1u));
  }
};

// N codes of WIDTH bits from an arbitrary bit of a shared-memory stream (the
// Med3x layout: a token's codes start wherever its coded offset puts them).
// get(i) reads code i at a compile-time position; get_dyn(j) a runtime one
// (code j of the run after flagged chunks were skipped) through a select
// chain over the loaded words (no local memory).
template <int N, int WIDTH>
struct CodeRunDyn {
  static constexpr int kNW = (31 + N * WIDTH + 31) / 32;
  uint32_t r[kNW];
  __device__ __forceinline__ void load(const uint32_t* __restrict__ s, uint32_t bit) {
    const uint32_t* p = s + (bit >> 5);
    const uint32_t sh = bit & 31;
    uint32_t w[kNW + 1];
#pragma unroll
    for (int i = 0; i < kNW; ++i) w[i] = p[i];
    w[kNW] = 0u;
#pragma unroll
    for (int i = 0; i < kNW; ++i) r[i] = __funnelshift_r(w[i], w[i + 1], sh);
  }
  __device__ __forceinline__ uint32_t get(int i) const {
    const int b = i * WIDTH, wi = b >> 5, sh = b & 31;
    uint32_t v = sh == 0 ? r[wi] : __funnelshift_r(r[wi], wi + 1 < kNW ? r[wi + 1] : 0u, sh);
    return WIDTH == 32 ? v : (v & ((1u << WIDTH) - 1u));
  }
  __device__ __forceinline__ uint32_t get_dyn(int j) const {
    const uint32_t b = (uint32_t)j * WIDTH, wi = b >> 5, sh = b & 31;
    uint32_t lo = r[0], hi = kNW > 1 ? r[1] : 0u;
#pragma unroll
    for (int i = 1; i < kNW; ++i)
      if (wi == (uint32_t)i) {
        lo = r[i];
        hi = i + 1 < kNW ? r[i + 1] : 0u;
      }
    const uint32_t v = __funnelshift_r(lo, hi, sh);
    return WIDTH == 32 ? v : (v & ((1u << WIDTH) - 1u));
  }
};

// split-KV merge of per-(row, part) partial (m, l, O) (attention.cu)
__global__ void combine_kernel(AttParams p);

}  // namespace hqmq
