// Fused HQMQ decode-inside-attention for sm_100a (split-KV / flash-decoding).
//
// Reference path replaced: attention.fused_attend (attention.py:137-199) —
// online softmax over KV tiles that are decoded in place; grouped queries
// (query head h reads kv head h // group, attention.py:29-69) and the
// decode-time causal offset (key j visible to query i iff j <= i + Tkv - Tq).
//
// Grid: (splits, batch * kv_heads, row_groups).  A CTA owns up to kRows query
// rows (the group's query heads x query tokens) of one kv head and a
// contiguous KV range.  Per 32-token tile it decodes K and V straight from the
// packed section streams into shared memory (codeword gather from the smem
// joint tables, radius from the fp16 scale), so dense K/V never touch HBM;
// then one thread per (row, token) forms the logit, a warp per row runs the
// online-softmax update, and one thread per (row, 4-dim chunk) accumulates
// P.V.  Partial (m, l, o) per split are merged by combine_kernel.
#include <algorithm>
#include <cstdint>
#include <cfloat>
#include <cmath>
#include <cstdlib>

#include "attention.cuh"

namespace hqmq {

constexpr int kAttThreads = 128;
constexpr int kKT = 32;          // keys per tile
constexpr int kRows = 4;         // query rows per CTA (one warp each)
constexpr int kMaxC = 32;        // head_dim <= 128
constexpr int kKStride = 4 * kMaxC + 4;  // padded smem row (floats)


__device__ __forceinline__ float4 decode_chunk(const AttView& v, const float4* tab, int64_t tok,
                                               int C, int c, int w, int br, int ncw, float rtop) {
  const uint64_t g = (uint64_t)tok * C + c;
  uint64_t pos = g;
  bool fl = false;
  if (v.flagw) {
    fl = (__ldg(v.flagw + (g >> 5)) >> (g & 31)) & 1u;
    uint64_t b = (uint64_t)tok * C;
    uint32_t nflag = 0;
    while (b < g) {
      const uint32_t word = __ldg(v.flagw + (b >> 5));
      const uint32_t sh = (uint32_t)(b & 31);
      const uint64_t take = min((uint64_t)(32 - sh), g - b);
      const uint32_t m = take == 32 ? 0xffffffffu : ((1u << take) - 1u);
      nflag += __popc((word >> sh) & m);
      b += take;
    }
    pos = (uint64_t)__ldg(v.tokoff + tok) + (uint64_t)(c - (int)nflag);
  }
  if (fl) {
    const ushort4 hv = __ldg(reinterpret_cast<const ushort4*>(v.payloads) + (g - pos));
    return make_float4(__half2float(__ushort_as_half(hv.x)), __half2float(__ushort_as_half(hv.y)),
                       __half2float(__ushort_as_half(hv.z)), __half2float(__ushort_as_half(hv.w)));
  }
  uint32_t idx = read_bits(v.idxw, pos * (uint64_t)w, w);
  const uint32_t q = read_bits(v.radw, pos * (uint64_t)br, br);
  idx = idx < (uint32_t)ncw ? idx : 0u;
  const float sig = __half2float(__ushort_as_half(__ldg(v.scales + tok)));
  const float rad = ((float)q * sig) * rtop;
  const float4 cw = tab[idx];
  return make_float4(rad * cw.x, rad * cw.y, rad * cw.z, rad * cw.w);
}

template <bool kSmemTab>
__global__ void __launch_bounds__(kAttThreads) attention_split_kernel(AttParams p) {
  extern __shared__ float4 dyn[];
  __shared__ __align__(16) float q_s[kRows][4 * kMaxC];
  __shared__ __align__(16) float k_s[kKT][kKStride];
  __shared__ __align__(16) float v_s[kKT][4 * kMaxC];
  __shared__ float p_s[kRows][kKT];
  __shared__ float alpha_s[kRows];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t bh = blockIdx.y;  // b * Hkv + hkv
  const int64_t b = (uint32_t)bh / (uint32_t)p.Hkv, hkv = (uint32_t)bh % (uint32_t)p.Hkv;  // (32-bit)
  const int split = blockIdx.x;
  const int row0 = blockIdx.z * kRows;
  const int C = p.C, D = (int)p.D, ncw = kGroupOrder * p.S;
  const float rtop = 1.0f / (float)((1 << p.br) - 1);

  const float4* ktab = p.k.table + hkv * ncw;
  const float4* vtab = p.v.table + hkv * ncw;
  if (kSmemTab) {
    float4* kt = dyn;
    float4* vt = dyn + ncw;
    for (int i = tid; i < ncw; i += kAttThreads) {
      kt[i] = __ldg(ktab + i);
      vt[i] = __ldg(vtab + i);
    }
    ktab = kt;
    vtab = vt;
  }
  // query rows (pre-scaled by softmax scale * log2 e)
  for (int i = tid; i < kRows * D; i += kAttThreads) {
    const int r = i / D, d = i - r * D;
    const int rr = row0 + r;
    float val = 0.f;
    if (rr < p.nrows) {
      const int gi = rr / (int)p.Tq, qi = rr - gi * (int)p.Tq;
      const int64_t hq = hkv * p.g + gi;
      val = p.q[((b * p.Hq + hq) * p.Tq + qi) * p.D + d] * p.scale_log2;
    }
    q_s[r][d] = val;
  }
  const int64_t kbeg = (int64_t)split * p.keys_per_split;
  const int64_t kend = min(p.Tkv, kbeg + p.keys_per_split);
  // row state (one warp per row): running max m (log2 domain) and sum l
  float m_run = -INFINITY, l_run = 0.f;
  // accumulators: thread = (row r = warp, chunk c = lane) [+32 for C > 32 not supported]
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  const int my_row = row0 + warp;
  int64_t vis = p.Tkv;  // keys visible to my row: j < vis
  if (my_row < p.nrows && p.causal) {
    const int qi = my_row % (int)p.Tq;
    vis = qi + (p.Tkv - p.Tq) + 1;
  }
  __syncthreads();

  for (int64_t t0 = kbeg; t0 < kend; t0 += kKT) {
    const int nt = (int)min((int64_t)kKT, kend - t0);
    // ---- decode K/V tile into smem (warp w: tokens w, w+4, ...; lane: chunk)
    for (int tt = warp; tt < nt; tt += kAttThreads / 32) {
      const int64_t tok = (b * p.Hkv + hkv) * p.Tkv + t0 + tt;
      if (lane < C) {
        const float4 kc = decode_chunk(p.k, ktab, tok, C, lane, p.w, p.br, ncw, rtop);
        const float4 vc = decode_chunk(p.v, vtab, tok, C, lane, p.w, p.br, ncw, rtop);
        *reinterpret_cast<float4*>(&k_s[tt][4 * lane]) = kc;
        *reinterpret_cast<float4*>(&v_s[tt][4 * lane]) = vc;
      }
    }
    __syncthreads();
    // ---- logits: warp = row, lane = key
    float s = -INFINITY;
    if (my_row < p.nrows && lane < nt && t0 + lane < vis) {
      float a0 = 0.f, a1 = 0.f;
      for (int c = 0; c < C; ++c) {
        const float4 kk = *reinterpret_cast<const float4*>(&k_s[lane][4 * c]);
        const float4 qq = *reinterpret_cast<const float4*>(&q_s[warp][4 * c]);
        a0 = fmaf(qq.x, kk.x, a0);
        a1 = fmaf(qq.y, kk.y, a1);
        a0 = fmaf(qq.z, kk.z, a0);
        a1 = fmaf(qq.w, kk.w, a1);
      }
      s = a0 + a1;
    }
    const float tmax = warp_max(s);
    const float m_new = fmaxf(m_run, tmax);
    float pr = 0.f, alpha = 1.f;
    if (m_new != -INFINITY) {
      pr = s == -INFINITY ? 0.f : exp2f(s - m_new);
      alpha = m_run == -INFINITY ? 0.f : exp2f(m_run - m_new);
    }
    float psum = pr;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) psum += __shfl_xor_sync(0xffffffffu, psum, o);
    l_run = l_run * alpha + psum;
    m_run = m_new;
    p_s[warp][lane] = pr;
    __syncwarp();
    // ---- P.V: warp = row, lane = 4-dim chunk
    if (lane < C) {
      acc.x *= alpha; acc.y *= alpha; acc.z *= alpha; acc.w *= alpha;
      for (int tt = 0; tt < nt; ++tt) {
        const float pv = p_s[warp][tt];
        const float4 vv = *reinterpret_cast<const float4*>(&v_s[tt][4 * lane]);
        acc.x = fmaf(pv, vv.x, acc.x);
        acc.y = fmaf(pv, vv.y, acc.y);
        acc.z = fmaf(pv, vv.z, acc.z);
        acc.w = fmaf(pv, vv.w, acc.w);
      }
    }
    __syncthreads();
  }
  (void)alpha_s;
  if (my_row >= p.nrows) return;
  if (p.splits == 1) {
    if (lane < C) {
      const int gi = my_row / (int)p.Tq, qi = my_row - gi * (int)p.Tq;
      const int64_t hq = hkv * p.g + gi;
      float* o = p.out + ((b * p.Hq + hq) * p.Tq + qi) * p.D + 4 * lane;
      const float inv = 1.0f / l_run;
      *reinterpret_cast<float4*>(o) = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    }
    return;
  }
  const int64_t pr_idx = (bh * p.nrows + my_row) * p.splits + split;
  if (lane < C)
    *reinterpret_cast<float4*>(p.part_o + pr_idx * p.D + 4 * lane) = acc;
  if (lane == 0) {
    p.part_ml[2 * pr_idx] = m_run;
    p.part_ml[2 * pr_idx + 1] = l_run;
  }
}

__global__ void combine_kernel(AttParams p) {
  const int64_t bh = blockIdx.x;
  const int r = blockIdx.y;
  const int64_t b = (uint32_t)bh / (uint32_t)p.Hkv, hkv = (uint32_t)bh % (uint32_t)p.Hkv;  // (32-bit)
  const int64_t base = (bh * p.nrows + r) * p.splits;
  float M = -INFINITY;
  for (int s = 0; s < p.splits; ++s) M = fmaxf(M, p.part_ml[2 * (base + s)]);
  float L = 0.f;
  for (int s = 0; s < p.splits; ++s) {
    const float m = p.part_ml[2 * (base + s)];
    if (m != -INFINITY) L += p.part_ml[2 * (base + s) + 1] * exp2f(m - M);
  }
  const int gi = r / (int)p.Tq, qi = r - gi * (int)p.Tq;
  const int64_t hq = hkv * p.g + gi;
  float* o = p.out + ((b * p.Hq + hq) * p.Tq + qi) * p.D;
  for (int d = threadIdx.x; d < p.D; d += blockDim.x) {
    float acc = 0.f;
    for (int s = 0; s < p.splits; ++s) {
      const float m = p.part_ml[2 * (base + s)];
      if (m != -INFINITY) acc += p.part_o[(base + s) * p.D + d] * exp2f(m - M);
    }
    o[d] = acc * p.o_scale / L;
  }
}

// ------------------------------------------------------------------------
// fp64 path: fused_attend(dtype=float64), the reference's default contract
// (attention.py:137-199, held to 1e-10 of the dense fp64 attention by
// test_attention.py:83-87).  K/V are decoded exactly as decode_token_range
// does (codec.py:315-325: ((q * sigma_w) / top) * codeword in fp64, payload
// rows widened from fp16), logits, softmax (exp) and P.V run in fp64 on the
// CUDA cores.  Same CTA geometry as attention_split_kernel: 4 query rows (one
// warp each) of one kv head x a key range, 32-key tiles decoded into shared
// memory once for the 4 rows; partial (m, l, o) per split merged by
// combine_f64_kernel.  Any head_dim <= 128 (multiple of 4), Med3x included.
constexpr int kF64Stride = 129;  // doubles per smem K row: lane = key reads conflict-free

__device__ __forceinline__ void decode_chunk_f64(const AttView& v, const double* tab, int64_t tok,
                                                 int C, int c, int w, int br, int ncw, double top,
                                                 double (&x)[4]) {
  const uint64_t g = (uint64_t)tok * C + c;
  uint64_t pos = g;
  bool fl = false;
  if (v.flagw) {
    fl = (__ldg(v.flagw + (g >> 5)) >> (g & 31)) & 1u;
    uint64_t b = (uint64_t)tok * C;
    uint32_t nflag = 0;
    while (b < g) {
      const uint32_t word = __ldg(v.flagw + (b >> 5));
      const uint32_t sh = (uint32_t)(b & 31);
      const uint64_t take = min((uint64_t)(32 - sh), g - b);
      const uint32_t m = take == 32 ? 0xffffffffu : ((1u << take) - 1u);
      nflag += __popc((word >> sh) & m);
      b += take;
    }
    pos = (uint64_t)__ldg(v.tokoff + tok) + (uint64_t)(c - (int)nflag);
  }
  if (fl) {
    const ushort4 hv = __ldg(reinterpret_cast<const ushort4*>(v.payloads) + (g - pos));
    x[0] = (double)__half2float(__ushort_as_half(hv.x));
    x[1] = (double)__half2float(__ushort_as_half(hv.y));
    x[2] = (double)__half2float(__ushort_as_half(hv.z));
    x[3] = (double)__half2float(__ushort_as_half(hv.w));
    return;
  }
  uint32_t idx = read_bits(v.idxw, pos * (uint64_t)w, w);
  const uint32_t q = read_bits(v.radw, pos * (uint64_t)br, br);
  idx = idx < (uint32_t)ncw ? idx : 0u;
  const double sw = (double)__half2float(__ushort_as_half(__ldg(v.scales + tok)));
  const double rad = __ddiv_rn(__dmul_rn((double)q, sw), top);
#pragma unroll
  for (int i = 0; i < 4; ++i) x[i] = __dmul_rn(rad, __ldg(tab + 4 * (int64_t)idx + i));
}

struct AttParams64 {
  const double* q;
  double* out;
  double* part_o;   // [B*Hkv][rows][splits][D]
  double* part_ml;  // [B*Hkv][rows][splits][2]
  double scale;
};

__global__ void __launch_bounds__(kAttThreads) attention_f64_kernel(AttParams p, AttParams64 p64) {
  extern __shared__ __align__(16) double dsm[];
  double* q_s = dsm;                          // [kRows][128]
  double* k_s = q_s + kRows * 4 * kMaxC;      // [kKT][kF64Stride]
  double* v_s = k_s + kKT * kF64Stride;       // [kKT][128]
  double* p_s = v_s + kKT * 4 * kMaxC;        // [kRows][kKT]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t bh = blockIdx.y;
  const int64_t b = (uint32_t)bh / (uint32_t)p.Hkv, hkv = (uint32_t)bh % (uint32_t)p.Hkv;  // (32-bit)
  const int split = blockIdx.x;
  const int row0 = blockIdx.z * kRows;
  const int C = p.C, D = (int)p.D, ncw = kGroupOrder * p.S;
  const double top = (double)((1 << p.br) - 1);
  const double* ktab = p.k.table64 + (int64_t)hkv * ncw * 4;
  const double* vtab = p.v.table64 + (int64_t)hkv * ncw * 4;
  for (int i = tid; i < kRows * 4 * kMaxC; i += kAttThreads) {
    const int r = i / (4 * kMaxC), d = i - r * 4 * kMaxC;
    const int rr = row0 + r;
    double val = 0.0;
    if (rr < p.nrows && d < D) {
      const int gi = rr / (int)p.Tq, qi = rr - gi * (int)p.Tq;
      const int64_t hq = hkv * p.g + gi;
      val = p64.q[((b * p.Hq + hq) * p.Tq + qi) * p.D + d];
    }
    q_s[i] = val;
  }
  const int64_t kbeg = (int64_t)split * p.keys_per_split;
  const int64_t kend = min(p.Tkv, kbeg + p.keys_per_split);
  double m_run = -INFINITY, l_run = 0.0;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  const int my_row = row0 + warp;
  int64_t vis = p.Tkv;
  if (my_row < p.nrows && p.causal) vis = (my_row % (int)p.Tq) + (p.Tkv - p.Tq) + 1;
  __syncthreads();
  for (int64_t t0 = kbeg; t0 < kend; t0 += kKT) {
    const int nt = (int)min((int64_t)kKT, kend - t0);
    for (int i = tid; i < nt * C; i += kAttThreads) {
      const int tt = i / C, c = i - tt * C;
      const int64_t tok = (b * p.Hkv + hkv) * p.Tkv + t0 + tt;
      double x[4];
      decode_chunk_f64(p.k, ktab, tok, C, c, p.w, p.br, ncw, top, x);
#pragma unroll
      for (int e = 0; e < 4; ++e) k_s[tt * kF64Stride + 4 * c + e] = x[e];
      decode_chunk_f64(p.v, vtab, tok, C, c, p.w, p.br, ncw, top, x);
#pragma unroll
      for (int e = 0; e < 4; ++e) v_s[tt * 4 * kMaxC + 4 * c + e] = x[e];
    }
    __syncthreads();
    // logits (attention.py:176): (q . k) * scale, lane = key
    double s = -INFINITY;
    if (my_row < p.nrows && lane < nt && t0 + lane < vis) {
      const double* kr = k_s + lane * kF64Stride;
      const double* qr = q_s + warp * 4 * kMaxC;
      double a0 = 0.0, a1 = 0.0;
      for (int d = 0; d < 4 * C; d += 2) {
        a0 = fma(qr[d], kr[d], a0);
        a1 = fma(qr[d + 1], kr[d + 1], a1);
      }
      s = (a0 + a1) * p64.scale;
    }
    double tmax = s;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tmax = fmax(tmax, __shfl_xor_sync(0xffffffffu, tmax, o));
    const double m_new = fmax(m_run, tmax);
    double pr = 0.0, alpha = 1.0;
    if (m_new != -INFINITY) {
      pr = s == -INFINITY ? 0.0 : exp(s - m_new);
      alpha = m_run == -INFINITY ? 0.0 : exp(m_run - m_new);
    }
    double psum = pr;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) psum += __shfl_xor_sync(0xffffffffu, psum, o);
    l_run = l_run * alpha + psum;
    m_run = m_new;
    p_s[warp * kKT + lane] = pr;
    __syncwarp();
    if (lane < C) {
#pragma unroll
      for (int e = 0; e < 4; ++e) acc[e] *= alpha;
      for (int tt = 0; tt < nt; ++tt) {
        const double pv = p_s[warp * kKT + tt];
        const double* vr = v_s + tt * 4 * kMaxC + 4 * lane;
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[e] = fma(pv, vr[e], acc[e]);
      }
    }
    __syncthreads();
  }
  if (my_row >= p.nrows || lane >= C) return;
  const int gi = my_row / (int)p.Tq, qi = my_row - gi * (int)p.Tq;
  const int64_t hq = hkv * p.g + gi;
  if (p.splits == 1) {
    double* o = p64.out + ((b * p.Hq + hq) * p.Tq + qi) * p.D + 4 * lane;
#pragma unroll
    for (int e = 0; e < 4; ++e) o[e] = acc[e] / l_run;
    return;
  }
  const int64_t pr_idx = (bh * p.nrows + my_row) * p.splits + split;
#pragma unroll
  for (int e = 0; e < 4; ++e) p64.part_o[pr_idx * p.D + 4 * lane + e] = acc[e];
  if (lane == 0) {
    p64.part_ml[2 * pr_idx] = m_run;
    p64.part_ml[2 * pr_idx + 1] = l_run;
  }
}

__global__ void combine_f64_kernel(AttParams p, AttParams64 p64) {
  const int64_t bh = blockIdx.x;
  const int r = blockIdx.y;
  const int64_t b = (uint32_t)bh / (uint32_t)p.Hkv, hkv = (uint32_t)bh % (uint32_t)p.Hkv;  // (32-bit)
  const int64_t base = (bh * p.nrows + r) * p.splits;
  double M = -INFINITY;
  for (int s = 0; s < p.splits; ++s) M = fmax(M, p64.part_ml[2 * (base + s)]);
  double L = 0.0;
  for (int s = 0; s < p.splits; ++s) {
    const double m = p64.part_ml[2 * (base + s)];
    if (m != -INFINITY) L += p64.part_ml[2 * (base + s) + 1] * exp(m - M);
  }
  const int gi = r / (int)p.Tq, qi = r - gi * (int)p.Tq;
  const int64_t hq = hkv * p.g + gi;
  double* o = p64.out + ((b * p.Hq + hq) * p.Tq + qi) * p.D;
  for (int d = threadIdx.x; d < p.D; d += blockDim.x) {
    double acc = 0.0;
    for (int s = 0; s < p.splits; ++s) {
      const double m = p64.part_ml[2 * (base + s)];
      if (m != -INFINITY) acc += p64.part_o[(base + s) * p.D + d] * exp(m - M);
    }
    o[d] = acc / L;
  }
}

__host__ inline size_t f64_smem_bytes() {
  return sizeof(double) *
         ((size_t)kRows * 4 * kMaxC + (size_t)kKT * kF64Stride + (size_t)kKT * 4 * kMaxC +
          (size_t)kRows * kKT);
}

// ------------------------------------------------------------------------
// Tensor-core fast path (head_dim 128, no outlier extraction, <= 8 query rows
// per kv head, i.e. decode with GQA group <= 8) — warp-independent
// flash-decoding inside the CTA, with K/V decoded straight into mma.sync
// operand registers (no fp16 K/V tile in shared memory):
//   * 128-key tiles of the K and V sections (index / radius words and fp16
//     scales) stream into a kMStages-deep shared ring with cp.async.bulk; a
//     full mbarrier per stage signals arrival, and the last warp to release a
//     stage (shared-memory counter) issues that stage's next tile;
//   * consumer warp w owns keys [16w, 16w+16) of every tile.  QK^T and PV are
//     sums over head dims, so any permutation of the dims applied to both
//     operands (and undone when O is written) leaves them unchanged.  The
//     permutations below make every mma fragment element come from ONE
//     decoded 4-dim chunk, so each (key, chunk) is decoded exactly once, by
//     the lane whose fragment needs it:
//       S = Q K^T  (m16n8k16, M = query rows, N = 8 keys, K = 16 dims):
//         lane (g, t) holds B[k = 2t, 2t+1, 2t+8, 2t+9][key g]; k-slab ks maps
//         those 4 positions to chunk 8t + ks  ->  the lane decodes chunks
//         8t..8t+7 of key g (one contiguous run of 8 codes per stream);
//       O^T += V^T P^T (M = 16 dims, N = query rows, K = 16 keys):
//         lane (g, t) holds A[m = g, g+8][k = 2t, 2t+1, 2t+8, 2t+9]; m-tiles
//         (2j, 2j+1) map (m = g, g+8) to elements (0, 1) / (2, 3) of chunk
//         4g + j  ->  the lane decodes chunks 4g..4g+3 of keys 2t, 2t+1,
//         2t+8, 2t+9;
//     P^T's B fragments are the S accumulators themselves (S->P register
//     reuse), with the per-key scale sigma/top folded into S (K) and P (V);
//   * the warps' (m, l, O) are merged through shared memory at the end.
constexpr int kMT = 128;          // keys per CTA tile (8 warps x 16)
constexpr int kMStages = 4;
constexpr int kMConsumers = 8;
constexpr int kMThreads = kMConsumers * 32;

struct RingGeom {
  uint32_t ki, kr, ks, vi, vr, vs, kf, ka, vf, va, kp, vp, bytes;
};
// outlier payload rows a Med3x stage holds per tensor (the tile's rows are one
// contiguous range of the payload section; beyond this, global loads)
constexpr int kPayRows = 256;

// One ring stage: K and V index / radius words and fp16 scales of a 128-key
// tile; with Med3x (kFlags) also each key's flag word and its aux word (the
// token's coded offset in the contiguous layout, its payload row in the paged
// one), and slack for the 16-byte-aligned start of a compact code range.
__host__ __device__ inline RingGeom ring_geom(int w, int br, bool flags = false) {
  // (the Med3x stage packs its regions at 16 bytes, the bulk-copy alignment,
  // so that two CTAs still fit an SM at S = 64)
  const uint32_t al = flags ? 16u : 128u;
  auto up = [al](uint32_t x) { return (x + al - 1u) / al * al; };
  const uint32_t slack = flags ? 64u : 16u;
  RingGeom g;
  uint32_t o = 0;
  g.ki = o; o += up(kMT * w * 4 + slack);
  g.kr = o; o += up(kMT * br * 4 + slack);
  g.ks = o; o += up(kMT * 2);
  g.vi = o; o += up(kMT * w * 4 + slack);
  g.vr = o; o += up(kMT * br * 4 + slack);
  g.vs = o; o += up(kMT * 2);
  g.kf = g.ka = g.vf = g.va = g.kp = g.vp = 0;
  if (flags) {
    g.kf = o; o += kMT * 4;
    g.ka = o; o += kMT * 4;
    g.vf = o; o += kMT * 4;
    g.va = o; o += kMT * 4;
    g.kp = o; o += (kPayRows + 2) * 8;
    g.vp = o; o += (kPayRows + 2) * 8;
  }
  g.bytes = o;
  return g;
}

// Med3x extras after the ring: Q rows in fp32 (pre-scaled, natural dim order)
// for the outlier-chunk score corrections, and per-warp P tiles for the
// outlier-chunk PV corrections.
constexpr size_t kFlagExtra = (size_t)8 * 128 * 4 + (size_t)kMConsumers * 8 * 16 * 4 + 8 * 32 * 8;

constexpr size_t kMaxDynSmem = 220 * 1024;  // under sm_100's 227 KB per CTA, static shared memory included
constexpr int kMStagesFlags = 2;  // Med3x ring depth (room for the residual tables)

__host__ __device__ inline size_t mma_smem_bytes(int S, int w, int br, bool flags = false) {
  const size_t tab = (flags ? 4 : 2) * (size_t)kGroupOrder * S * 8;
  const size_t ring = (flags ? kMStagesFlags : kMStages) * (size_t)ring_geom(w, br, flags).bytes;
  const size_t merge = (size_t)kMConsumers * 8 * 130 * 4;  // O + (m, l) per warp/row
  return tab + (ring > merge ? ring : merge) + (flags ? kFlagExtra : 0);
}

// Med3x (kFlags): flagged chunks carry no code; their fp16 payload row is the
// value.  The MMAs see them as zero (radius code forced to 0) and each is
// added in fp32 on the CUDA cores: q . payload into the score of its key
// (lane-local: the S-accumulator lane of (row, key) does it) and
// p(row, key) * payload into O (the O^T lane owning the chunk's dims, with P
// from a per-warp shared tile).  Codes of the unflagged chunks are found from
// the key's coded offset (contiguous: token_offsets; paged: fixed slots).
template <int W, int BR, bool kPaged = false, bool kFlags = false>
__global__ void __launch_bounds__(kMThreads, 2) attention_mma_kernel(AttParams p) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) uint64_t full[kMStages];
  __shared__ __align__(8) uint64_t tab_bar;
  __shared__ unsigned int released[kMStages];
  // Med3x, contiguous layout: first staged payload row and staged row count
  // per stage and tensor (count 0: global loads)
  __shared__ unsigned long long pay_base[kFlags ? kMStages : 1][2];
  __shared__ uint32_t pay_n[kFlags ? kMStages : 1][2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int ncw = kGroupOrder * p.S;
  constexpr int w = W, br = BR;
  constexpr int NS = kFlags ? kMStagesFlags : kMStages;  // ring depth
  // Med3x: tables are converted in-kernel (V needs its fp16 hi / lo pair)
  const bool tab_tma = !kFlags && p.k.table16 != nullptr && p.v.table16 != nullptr;
  const RingGeom gm = ring_geom(w, br, kFlags);
  uint2* ktab = reinterpret_cast<uint2*>(sm);
  uint2* vtab = ktab + ncw;
  // Med3x: fp16 residual tables cw - fp16(cw) of K and V (split-fp16 S and P V)
  uint2* vtab_lo = vtab + ncw;
  uint2* ktab_lo = vtab + 2 * ncw;
  unsigned char* ring = reinterpret_cast<unsigned char*>(vtab + (kFlags ? 3 : 1) * ncw);
  // Med3x extras (kFlags only): after the ring (or the merge area)
  float* qs = nullptr;   // [8][128] fp32, scale_log2 folded in
  float* pws = nullptr;  // [warp][8 rows][16 keys]
  uint2* qlo_s = nullptr;  // [ks][lane]: fp16 residual of the Q A-fragments
  if constexpr (kFlags) {
    const size_t rb = NS * (size_t)gm.bytes, mb = (size_t)kMConsumers * 8 * 130 * 4;
    qs = reinterpret_cast<float*>(ring + (rb > mb ? rb : mb));
    pws = qs + 8 * 128;
    qlo_s = reinterpret_cast<uint2*>(pws + kMConsumers * 128);
  }

  const int64_t bh = blockIdx.y;
  const int64_t b = (uint32_t)bh / (uint32_t)p.Hkv, hkv = (uint32_t)bh % (uint32_t)p.Hkv;  // (32-bit)
  const int64_t kbeg = (int64_t)blockIdx.x * p.keys_per_split;
  const int64_t tkv = kPaged ? (int64_t)__ldg(p.kv_lens + b) : p.Tkv;  // this sequence's keys
  const int64_t kend = min(tkv, kbeg + p.keys_per_split);
  const int64_t ntile = kend > kbeg ? ceil_div(kend - kbeg, kMT) : 0;
  const int64_t tokrow = bh * p.Tkv;

  if (tid == 0) {
    for (int s = 0; s < NS; ++s) {
      mbar_init(&full[s], 1);
      released[s] = 0u;
    }
    mbar_init(&tab_bar, 1);
    fence_mbar_init();
  }
  __syncthreads();

  // first 16-byte-aligned word of a compact code range starting at code c0
  auto range_lo = [](uint64_t c0, int width) -> uint64_t { return ((c0 * width) >> 5) & ~3ull; };
  auto issue = [&](int64_t k, int stage) {
    int64_t t = tokrow + kbeg + k * kMT;
    int ntok = (int)min((int64_t)kMT, kend - (kbeg + k * kMT));
    if constexpr (kPaged) {  // tile = one whole page (keys past kend are masked)
      t = (int64_t)__ldg(p.block_table + bh * p.max_pages + (kbeg + k * kMT) / kMT) * kMT;
      ntok = kMT;
    }
    unsigned char* s = ring + (size_t)stage * gm.bytes;
    const uint32_t sb = ntok * 2;
    if constexpr (kFlags && !kPaged) {
      // compact streams: the tile's codes are [c0, c1) of the coded order
      const uint32_t fb = ntok * 4;  // ntok % 8 == 0 (T_kv % 8 == 0): 16-byte multiple
      uint32_t ib[2], rbb[2], pb[2];
      uint64_t iw0[2], rw0[2], pa0[2];
      const AttView* vw[2] = {&p.k, &p.v};
#pragma unroll
      for (int r = 0; r < 2; ++r) {
        const uint64_t c0 = __ldg(vw[r]->tokoff + t);
        const uint64_t cl = __ldg(vw[r]->tokoff + t + ntok - 1);
        const uint32_t fl_last = __ldg(vw[r]->flagw + t + ntok - 1);
        const uint64_t c1 = cl + 32u - (uint64_t)__popc(fl_last);
        iw0[r] = range_lo(c0, w);
        rw0[r] = range_lo(c0, br);
        ib[r] = (uint32_t)((((c1 * w + 31) >> 5) - iw0[r] + 3) & ~3ull) * 4u;
        rbb[r] = (uint32_t)((((c1 * br + 31) >> 5) - rw0[r] + 3) & ~3ull) * 4u;
        // the tile's payload rows [t*32 - c0, (t+ntok-1)*32 - cl + flagged(last))
        const uint64_t p0 = (uint64_t)t * 32u - c0;
        const uint64_t p1 = (uint64_t)(t + ntok - 1) * 32u - cl + (uint64_t)__popc(fl_last);
        pa0[r] = p0 & ~1ull;
        const uint64_t pa1 = (p1 + 1) & ~1ull;
        const bool st = p1 > p0 && pa1 - pa0[r] <= (uint64_t)kPayRows + 2;
        pb[r] = st ? (uint32_t)(pa1 - pa0[r]) * 8u : 0u;
        pay_base[stage][r] = pa0[r];
        pay_n[stage][r] = st ? (uint32_t)(pa1 - pa0[r]) : 0u;
      }
      fence_proxy_async();
      mbar_arrive_expect_tx(&full[stage], ib[0] + rbb[0] + ib[1] + rbb[1] + 2 * (sb + 2 * fb) + pb[0] + pb[1]);
      if (pb[0]) bulk_g2s(s + gm.kp, p.k.payloads + pa0[0] * 4, pb[0], &full[stage]);
      if (pb[1]) bulk_g2s(s + gm.vp, p.v.payloads + pa0[1] * 4, pb[1], &full[stage]);
      bulk_g2s(s + gm.ki, p.k.idxw + iw0[0], ib[0], &full[stage]);
      bulk_g2s(s + gm.kr, p.k.radw + rw0[0], rbb[0], &full[stage]);
      bulk_g2s(s + gm.ks, p.k.scales + t, sb, &full[stage]);
      bulk_g2s(s + gm.kf, p.k.flagw + t, fb, &full[stage]);
      bulk_g2s(s + gm.ka, p.k.tokoff + t, fb, &full[stage]);
      bulk_g2s(s + gm.vi, p.v.idxw + iw0[1], ib[1], &full[stage]);
      bulk_g2s(s + gm.vr, p.v.radw + rw0[1], rbb[1], &full[stage]);
      bulk_g2s(s + gm.vs, p.v.scales + t, sb, &full[stage]);
      bulk_g2s(s + gm.vf, p.v.flagw + t, fb, &full[stage]);
      bulk_g2s(s + gm.va, p.v.tokoff + t, fb, &full[stage]);
      return;
    }
    const uint32_t ib = ntok * w * 4, rb = ntok * br * 4;
    const uint32_t fb = kFlags ? ntok * 4 : 0;
    fence_proxy_async();
    mbar_arrive_expect_tx(&full[stage], 2 * (ib + rb + sb + 2 * fb));
    bulk_g2s(s + gm.ki, p.k.idxw + t * w, ib, &full[stage]);
    bulk_g2s(s + gm.kr, p.k.radw + t * br, rb, &full[stage]);
    bulk_g2s(s + gm.ks, p.k.scales + t, sb, &full[stage]);
    bulk_g2s(s + gm.vi, p.v.idxw + t * w, ib, &full[stage]);
    bulk_g2s(s + gm.vr, p.v.radw + t * br, rb, &full[stage]);
    bulk_g2s(s + gm.vs, p.v.scales + t, sb, &full[stage]);
    if constexpr (kFlags) {  // paged Med3x: flag words and payload rows per token
      bulk_g2s(s + gm.kf, p.k.flagw + t, fb, &full[stage]);
      bulk_g2s(s + gm.ka, p.k.tokoff + t, fb, &full[stage]);
      bulk_g2s(s + gm.vf, p.v.flagw + t, fb, &full[stage]);
      bulk_g2s(s + gm.va, p.v.tokoff + t, fb, &full[stage]);
    }
  };
  // release a stage; the last of the 8 warps refills it with tile k + NS
  auto release = [&](int64_t k, int stage) {
    __syncwarp();  // every lane's reads of the stage precede lane 0's release
    if (lane == 0) {
      if (stage_release(&released[stage]) == kMConsumers - 1) {
        released[stage] = 0u;
        if (k + NS < ntile) issue(k + NS, stage);
      }
    }
  };
  // the first tiles stream in while the joint tables are converted to fp16
  if (tid == 0) {
    if (tab_tma) {  // fp16 tables by TMA, beside the first tiles
      const uint32_t tb = (uint32_t)ncw * 8u;
      fence_proxy_async();
      mbar_arrive_expect_tx(&tab_bar, 2 * tb);
      bulk_g2s(ktab, p.k.table16 + hkv * ncw, tb, &tab_bar);
      bulk_g2s(vtab, p.v.table16 + hkv * ncw, tb, &tab_bar);
    }
    for (int s = 0; s < NS && s < ntile; ++s) issue(s, s);
  }
  const int g4 = lane >> 2, t4 = lane & 3;  // mma fragment coordinates
  if constexpr (kFlags) {  // fp32 Q rows (natural dims) for the outlier corrections
    for (int i = tid; i < 8 * 128; i += kMThreads) {
      const int r = i >> 7, d = i & 127;
      float v = 0.f;
      if (r < p.nrows) {
        const int gi = r / (int)p.Tq, qi = r - gi * (int)p.Tq;
        v = __ldg(p.q + ((b * p.Hq + hkv * p.g + gi) * p.Tq + qi) * 128 + d) * p.scale_log2;
      }
      qs[i] = v;
    }
  }
  if (tab_tma) {
    mbar_wait(&tab_bar, 0u);
    if constexpr (kFlags) __syncthreads();
  } else {
    const float4* gk = p.k.table + hkv * ncw;
    const float4* gv = p.v.table + hkv * ncw;
    for (int i = tid; i < ncw; i += kMThreads) {
      const float4 a = __ldg(gk + i), c = __ldg(gv + i);
      const uint2 h = make_uint2(pack_half2(c.x, c.y), pack_half2(c.z, c.w));
      const uint2 hk = make_uint2(pack_half2(a.x, a.y), pack_half2(a.z, a.w));
      ktab[i] = hk;
      vtab[i] = h;
      if constexpr (kFlags) {
        const float2 h01 = __half22float2(*reinterpret_cast<const __half2*>(&h.x));
        const float2 h23 = __half22float2(*reinterpret_cast<const __half2*>(&h.y));
        vtab_lo[i] = make_uint2(pack_half2(c.x - h01.x, c.y - h01.y), pack_half2(c.z - h23.x, c.w - h23.y));
        const float2 k01 = __half22float2(*reinterpret_cast<const __half2*>(&hk.x));
        const float2 k23 = __half22float2(*reinterpret_cast<const __half2*>(&hk.y));
        ktab_lo[i] = make_uint2(pack_half2(a.x - k01.x, a.y - k01.y), pack_half2(a.z - k23.x, a.w - k23.y));
      }
    }
    __syncthreads();
  }

  const uint32_t cwmax = (uint32_t)ncw - 1u;
  float m_run = -INFINITY, l_run = 0.f;
  // O^T accumulators, m-tile 2j+h: c0/c1 = (dim 4(4g4+j)+2h, rows 2t4 / 2t4+1),
  // c2/c3 = (dim 4(4g4+j)+2h+1, rows 2t4 / 2t4+1)
  float oT[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) oT[i][0] = oT[i][1] = oT[i][2] = oT[i][3] = 0.f;

  // Q A-fragments (rows x permuted dims, rows 8..15 zero): k-slab ks holds
  // chunk 8*t4 + ks of row g4: qa[ks] = {elements 0,1 ; elements 2,3}
  uint32_t qa[8][2];
  const bool row_valid = g4 < p.nrows;
  {
    const int gi = row_valid ? g4 / (int)p.Tq : 0, qi = row_valid ? g4 - gi * (int)p.Tq : 0;
    const float4* qrow =
        reinterpret_cast<const float4*>(p.q + ((b * p.Hq + hkv * p.g + gi) * p.Tq + qi) * 128);
#pragma unroll
    for (int ks = 0; ks < 8; ++ks) {
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (row_valid) v = __ldg(qrow + 8 * t4 + ks);
      qa[ks][0] = pack_half2(v.x * p.scale_log2, v.y * p.scale_log2);
      qa[ks][1] = pack_half2(v.z * p.scale_log2, v.w * p.scale_log2);
      if constexpr (kFlags) {  // Q residual fragments (every warp holds the same Q)
        if (warp == 0) {
          const float2 h01 = __half22float2(*reinterpret_cast<const __half2*>(&qa[ks][0]));
          const float2 h23 = __half22float2(*reinterpret_cast<const __half2*>(&qa[ks][1]));
          qlo_s[ks * 32 + lane] = make_uint2(pack_half2(v.x * p.scale_log2 - h01.x, v.y * p.scale_log2 - h01.y),
                                             pack_half2(v.z * p.scale_log2 - h23.x, v.w * p.scale_log2 - h23.y));
        }
      }
    }
    if constexpr (kFlags) __syncthreads();
  }
  int64_t vis = tkv;  // keys j < vis are visible to row g4
  if (row_valid && p.causal) vis = (g4 % (int)p.Tq) + (tkv - p.Tq) + 1;
  const float rtop = 1.0f / (float)((1 << br) - 1);

  for (int64_t k = 0; k < ntile; ++k) {
    const int stage = (int)(k % NS);
    mbar_wait(&full[stage], (uint32_t)((k / NS) & 1));
    const unsigned char* s = ring + (size_t)stage * gm.bytes;
    const uint32_t* kiw = reinterpret_cast<const uint32_t*>(s + gm.ki);
    const uint32_t* krw = reinterpret_cast<const uint32_t*>(s + gm.kr);
    const uint16_t* ksc = reinterpret_cast<const uint16_t*>(s + gm.ks);
    const uint32_t* viw = reinterpret_cast<const uint32_t*>(s + gm.vi);
    const uint32_t* vrw = reinterpret_cast<const uint32_t*>(s + gm.vr);
    const uint16_t* vsc = reinterpret_cast<const uint16_t*>(s + gm.vs);
    const uint32_t* kfl = reinterpret_cast<const uint32_t*>(s + gm.kf);
    const uint32_t* kax = reinterpret_cast<const uint32_t*>(s + gm.ka);
    const uint32_t* vfl = reinterpret_cast<const uint32_t*>(s + gm.vf);
    const uint32_t* vax = reinterpret_cast<const uint32_t*>(s + gm.va);
    const int kw0 = warp * 16;                       // this warp's first key in the tile
    const int64_t t0 = kbeg + k * kMT + kw0;         // ... as a key index
    const int64_t tile_key0 = kbeg + k * kMT;
    // Med3x: bit base of the tile's compact ranges, the tile's first global token
    uint64_t kib0 = 0, krb0 = 0, vib0 = 0, vrb0 = 0;
    const int64_t gtok0 = tokrow + tile_key0;
    int nvalid = kMT;
    if constexpr (kFlags) {
      nvalid = (int)min((int64_t)kMT, kend - tile_key0);
      if constexpr (!kPaged) {
        kib0 = range_lo(kax[0], w) * 32u;
        krb0 = range_lo(kax[0], br) * 32u;
        vib0 = range_lo(vax[0], w) * 32u;
        vrb0 = range_lo(vax[0], br) * 32u;
      }
    }
    // flag word / payload row of a key of the tile (0 / unused past the valid keys)
    auto kflag = [&](int key) -> uint32_t { return key < nvalid ? kfl[key] : 0u; };
    auto vflag = [&](int key) -> uint32_t { return key < nvalid ? vfl[key] : 0u; };
    auto pay_row = [&](const uint32_t* ax, int key, uint32_t fw, int c) -> uint64_t {
      const uint64_t below = (uint64_t)__popc(fw & ((1u << c) - 1u));
      if constexpr (kPaged) return (uint64_t)ax[key] + below;
      return (uint64_t)(gtok0 + key) * 32u - (uint64_t)ax[key] + below;
    };
    // a payload row of tensor r (0 = K, 1 = V): from the stage when staged
    auto payload = [&](int r, uint64_t prow) -> ushort4 {
      if constexpr (!kPaged) {
        const uint64_t rel = prow - pay_base[stage][r];
        if (rel < pay_n[stage][r])
          return reinterpret_cast<const ushort4*>(s + (r ? gm.vp : gm.kp))[rel];
      }
      return __ldg(reinterpret_cast<const ushort4*>(r ? p.v.payloads : p.k.payloads) + prow);
    };
    if (t0 < kend) {
      // ---- S = Q K^T: lane decodes chunks 8*t4 .. 8*t4+7 of key kw0 + 8*nt + g4
      float sc[2][4];
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.f;
        const uint32_t key = (uint32_t)(kw0 + nt * 8 + g4);
        if constexpr (!kFlags) {
          CodeRun<8, W, 4> ic;
          CodeRun<8, BR, 4> rc;
          ic.load(kiw, key * 32u * W + (uint32_t)t4 * 8u * W);
          rc.load(krw, key * 32u * BR + (uint32_t)t4 * 8u * BR);
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const uint2 cw = ktab[min(ic.get(ks), cwmax)];
            const uint32_t qq = code_half2(rc.get(ks));
            mma_rows8(sc[nt], qa[ks][0], qa[ks][1], hmul2u(qq, cw.x), hmul2u(qq, cw.y));
          }
        } else {
          const uint32_t fk = kflag((int)key);
          const uint32_t lo = (uint32_t)t4 * 8u;
          const uint32_t frun = (fk >> lo) & 0xffu;
          uint32_t ibit, rbit;
          if constexpr (kPaged) {
            ibit = key * 32u * W + lo * W;
            rbit = key * 32u * BR + lo * BR;
          } else {
            const uint64_t c = (int)key < nvalid
                                   ? (uint64_t)kax[key] + lo - (uint64_t)__popc(fk & ((1u << lo) - 1u))
                                   : (uint64_t)kax[0];
            ibit = (uint32_t)(c * W - kib0);
            rbit = (uint32_t)(c * BR - krb0);
          }
          CodeRunDyn<8, W> ic;
          CodeRunDyn<8, BR> rc;
          ic.load(kiw, ibit);
          rc.load(krw, rbit);
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            uint32_t ci, cq;
            if constexpr (kPaged) {  // fixed slots: flagged codes are ignored
              ci = ic.get(ks);
              cq = (frun >> ks) & 1u ? 0u : rc.get(ks);
            } else if (frun == 0u) {
              ci = ic.get(ks);
              cq = rc.get(ks);
            } else {
              const int j = ks - __popc(frun & ((1u << ks) - 1u));
              const bool fl = (frun >> ks) & 1u;
              ci = fl ? 0u : ic.get_dyn(j);
              cq = fl ? 0u : rc.get_dyn(j);
            }
            // K = q * cw to ~fp32 as fp16 hi + lo; S += Qh Kh + Qh Kl + Ql Kh
            const uint2 ch = ktab[min(ci, cwmax)], cl = ktab_lo[min(ci, cwmax)];
            const float qf = (float)cq;
            const float2 h01 = __half22float2(*reinterpret_cast<const __half2*>(&ch.x));
            const float2 h23 = __half22float2(*reinterpret_cast<const __half2*>(&ch.y));
            const float2 l01 = __half22float2(*reinterpret_cast<const __half2*>(&cl.x));
            const float2 l23 = __half22float2(*reinterpret_cast<const __half2*>(&cl.y));
            const float k0 = qf * (h01.x + l01.x), k1 = qf * (h01.y + l01.y);
            const float k2 = qf * (h23.x + l23.x), k3 = qf * (h23.y + l23.y);
            const uint32_t kh0 = pack_half2(k0, k1), kh1 = pack_half2(k2, k3);
            const float2 r01 = __half22float2(*reinterpret_cast<const __half2*>(&kh0));
            const float2 r23 = __half22float2(*reinterpret_cast<const __half2*>(&kh1));
            const uint32_t kl0 = pack_half2(k0 - r01.x, k1 - r01.y);
            const uint32_t kl1 = pack_half2(k2 - r23.x, k3 - r23.y);
            const uint2 ql = qlo_s[ks * 32 + lane];
            mma_rows8(sc[nt], qa[ks][0], qa[ks][1], kh0, kh1);
            mma_rows8(sc[nt], qa[ks][0], qa[ks][1], kl0, kl1);
            mma_rows8(sc[nt], ql.x, ql.y, kh0, kh1);
          }
        }
      }
      // per-key scales sigma/top of this lane's 4 keys (2t4, 2t4+1, 2t4+8, 2t4+9)
      float kst[4], vst[4], sv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int kk = kw0 + (e >> 1) * 8 + t4 * 2 + (e & 1);
        const int64_t key = kbeg + k * kMT + kk;
        const bool in = key < kend;
        kst[e] = __half2float(__ushort_as_half(ksc[kk])) * rtop;
        vst[e] = in ? __half2float(__ushort_as_half(vsc[kk])) * rtop : 0.f;
        const bool ok = row_valid && in && key < vis;
        float corr = 0.f;
        if constexpr (kFlags) {  // outlier chunks of this key: q . payload in fp32
          const uint32_t fk = kflag(kk);
          uint32_t rem = fk;
          while (rem) {
            const int c = __ffs(rem) - 1;
            rem &= rem - 1u;
            const ushort4 hv = payload(0, pay_row(kax, kk, fk, c));
            const float4 qv = *reinterpret_cast<const float4*>(qs + g4 * 128 + 4 * c);
            corr += qv.x * __half2float(__ushort_as_half(hv.x)) +
                    qv.y * __half2float(__ushort_as_half(hv.y)) +
                    qv.z * __half2float(__ushort_as_half(hv.z)) +
                    qv.w * __half2float(__ushort_as_half(hv.w));
          }
        }
        sv[e] = ok ? sc[e >> 1][e & 1] * kst[e] + corr : -INFINITY;
      }
      // ---- online softmax for row g4 over this warp's 16 keys (log2 domain)
      float mx = fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3]));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
      const float m_new = fmaxf(m_run, mx);
      float pe[4], alpha = 1.f;
      if (m_new == -INFINITY) {
        pe[0] = pe[1] = pe[2] = pe[3] = 0.f;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) pe[e] = exp2f(sv[e] - m_new);
        alpha = exp2f(m_run - m_new);
      }
      float ps = (pe[0] + pe[1]) + (pe[2] + pe[3]);
      ps += __shfl_xor_sync(0xffffffffu, ps, 1);
      ps += __shfl_xor_sync(0xffffffffu, ps, 2);
      l_run = l_run * alpha + ps;
      m_run = m_new;
      // rescale: this thread's O^T columns are rows 2t4 and 2t4+1, whose
      // softmax state lives in lanes 8t4 and 8t4+4
      const float a_lo = __shfl_sync(0xffffffffu, alpha, t4 * 8);
      const float a_hi = __shfl_sync(0xffffffffu, alpha, t4 * 8 + 4);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        oT[i][0] *= a_lo; oT[i][1] *= a_hi; oT[i][2] *= a_lo; oT[i][3] *= a_hi;
      }
      // P^T B-fragments straight from the S accumulators, V scale folded in
      const uint32_t pb0 = pack_half2(pe[0] * vst[0], pe[1] * vst[1]);
      const uint32_t pb1 = pack_half2(pe[2] * vst[2], pe[3] * vst[3]);
      // ---- O^T += V^T P^T: lane decodes chunks 4*g4 .. 4*g4+3 of its 4 keys
      if constexpr (!kFlags) {
        uint2 vv[4][4];  // [key e][chunk j] -> 4 halves
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t key = (uint32_t)(kw0 + (e >> 1) * 8 + t4 * 2 + (e & 1));
          CodeRun<4, W, 8> ic;
          CodeRun<4, BR, 8> rc;
          ic.load(viw, key * 32u * W + (uint32_t)g4 * 4u * W);
          rc.load(vrw, key * 32u * BR + (uint32_t)g4 * 4u * BR);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint2 cw = vtab[min(ic.get(j), cwmax)];
            const uint32_t qq = code_half2(rc.get(j));
            vv[e][j] = make_uint2(hmul2u(qq, cw.x), hmul2u(qq, cw.y));
          }
        }
        release(k, stage);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          // m-tile 2j: (m = g4, g4+8) = elements (0, 1); m-tile 2j+1: elements (2, 3)
          // a0 = keys (2t4, 2t4+1) at m = g4 ; a1 = same keys at m = g4+8
          // a2 = keys (2t4+8, 2t4+9) at m = g4 ; a3 = same keys at m = g4+8
          const uint32_t x0 = vv[0][j].x, x1 = vv[1][j].x, x2 = vv[2][j].x, x3 = vv[3][j].x;
          const uint32_t y0 = vv[0][j].y, y1 = vv[1][j].y, y2 = vv[2][j].y, y3 = vv[3][j].y;
          mma_full(oT[2 * j], __byte_perm(x0, x1, 0x5410), __byte_perm(x0, x1, 0x7632),
                   __byte_perm(x2, x3, 0x5410), __byte_perm(x2, x3, 0x7632), pb0, pb1);
          mma_full(oT[2 * j + 1], __byte_perm(y0, y1, 0x5410), __byte_perm(y0, y1, 0x7632),
                   __byte_perm(y2, y3, 0x5410), __byte_perm(y2, y3, 0x7632), pb0, pb1);
        }
      } else {
        // Med3x: split-fp16 P and V (P = Ph + Pl, V = Vh + Vl, O += Vh Ph + Vl Ph +
        // Vh Pl): outlier caches give peaked softmax rows, where one fp16 V
        // rounding would show up at the 1e-3 level
        const float2 ph01 = __half22float2(*reinterpret_cast<const __half2*>(&pb0));
        const float2 ph23 = __half22float2(*reinterpret_cast<const __half2*>(&pb1));
        const uint32_t pl0 = pack_half2(pe[0] * vst[0] - ph01.x, pe[1] * vst[1] - ph01.y);
        const uint32_t pl1 = pack_half2(pe[2] * vst[2] - ph23.x, pe[3] * vst[3] - ph23.y);
        CodeRunDyn<4, W> icv[4];
        CodeRunDyn<4, BR> rcv[4];
        uint32_t frv[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const uint32_t key = (uint32_t)(kw0 + (e >> 1) * 8 + t4 * 2 + (e & 1));
          const uint32_t fv = vflag((int)key);
          const uint32_t lo = (uint32_t)g4 * 4u;
          frv[e] = (fv >> lo) & 0xfu;
          uint32_t ibit, rbit;
          if constexpr (kPaged) {
            ibit = key * 32u * W + lo * W;
            rbit = key * 32u * BR + lo * BR;
          } else {
            const uint64_t c = (int)key < nvalid
                                   ? (uint64_t)vax[key] + lo - (uint64_t)__popc(fv & ((1u << lo) - 1u))
                                   : (uint64_t)vax[0];
            ibit = (uint32_t)(c * W - vib0);
            rbit = (uint32_t)(c * BR - vrb0);
          }
          icv[e].load(viw, ibit);
          rcv[e].load(vrw, rbit);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          uint32_t hx[4], hy[4], lx[4], ly[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint32_t frun = frv[e];
            uint32_t ci, cq;
            if constexpr (kPaged) {
              ci = icv[e].get(j);
              cq = (frun >> j) & 1u ? 0u : rcv[e].get(j);
            } else if (frun == 0u) {
              ci = icv[e].get(j);
              cq = rcv[e].get(j);
            } else {
              const int jj = j - __popc(frun & ((1u << j) - 1u));
              const bool fl = (frun >> j) & 1u;
              ci = fl ? 0u : icv[e].get_dyn(jj);
              cq = fl ? 0u : rcv[e].get_dyn(jj);
            }
            const uint2 ch = vtab[min(ci, cwmax)], cl = vtab_lo[min(ci, cwmax)];
            const float qf = (float)cq;
            const float2 h01 = __half22float2(*reinterpret_cast<const __half2*>(&ch.x));
            const float2 h23 = __half22float2(*reinterpret_cast<const __half2*>(&ch.y));
            const float2 l01 = __half22float2(*reinterpret_cast<const __half2*>(&cl.x));
            const float2 l23 = __half22float2(*reinterpret_cast<const __half2*>(&cl.y));
            const float v0 = qf * (h01.x + l01.x), v1 = qf * (h01.y + l01.y);
            const float v2 = qf * (h23.x + l23.x), v3 = qf * (h23.y + l23.y);
            hx[e] = pack_half2(v0, v1);
            hy[e] = pack_half2(v2, v3);
            const float2 r01 = __half22float2(*reinterpret_cast<const __half2*>(&hx[e]));
            const float2 r23 = __half22float2(*reinterpret_cast<const __half2*>(&hy[e]));
            lx[e] = pack_half2(v0 - r01.x, v1 - r01.y);
            ly[e] = pack_half2(v2 - r23.x, v3 - r23.y);
          }
          mma_full(oT[2 * j], __byte_perm(hx[0], hx[1], 0x5410), __byte_perm(hx[0], hx[1], 0x7632),
                   __byte_perm(hx[2], hx[3], 0x5410), __byte_perm(hx[2], hx[3], 0x7632), pb0, pb1);
          mma_full(oT[2 * j], __byte_perm(lx[0], lx[1], 0x5410), __byte_perm(lx[0], lx[1], 0x7632),
                   __byte_perm(lx[2], lx[3], 0x5410), __byte_perm(lx[2], lx[3], 0x7632), pb0, pb1);
          mma_full(oT[2 * j], __byte_perm(hx[0], hx[1], 0x5410), __byte_perm(hx[0], hx[1], 0x7632),
                   __byte_perm(hx[2], hx[3], 0x5410), __byte_perm(hx[2], hx[3], 0x7632), pl0, pl1);
          mma_full(oT[2 * j + 1], __byte_perm(hy[0], hy[1], 0x5410), __byte_perm(hy[0], hy[1], 0x7632),
                   __byte_perm(hy[2], hy[3], 0x5410), __byte_perm(hy[2], hy[3], 0x7632), pb0, pb1);
          mma_full(oT[2 * j + 1], __byte_perm(ly[0], ly[1], 0x5410), __byte_perm(ly[0], ly[1], 0x7632),
                   __byte_perm(ly[2], ly[3], 0x5410), __byte_perm(ly[2], ly[3], 0x7632), pb0, pb1);
          mma_full(oT[2 * j + 1], __byte_perm(hy[0], hy[1], 0x5410), __byte_perm(hy[0], hy[1], 0x7632),
                   __byte_perm(hy[2], hy[3], 0x5410), __byte_perm(hy[2], hy[3], 0x7632), pl0, pl1);
        }
      }
      if constexpr (kFlags) {
        // ---- outlier V chunks: O[row][dims of chunk c] += p(row, key) * payload
        const uint32_t fvl = lane < 16 ? vflag(kw0 + lane) : 0u;
        if (__any_sync(0xffffffffu, fvl != 0u)) {
          float* pw = pws + warp * 128;  // [row][16 keys]
#pragma unroll
          for (int e = 0; e < 4; ++e) pw[g4 * 16 + (e >> 1) * 8 + t4 * 2 + (e & 1)] = pe[e];
          __syncwarp();
          for (int kk = 0; kk < 16; ++kk) {
            const uint32_t fv = vflag(kw0 + kk);
            uint32_t bits = (fv >> (4 * g4)) & 0xfu;
            if (!bits) continue;
            const float p0 = pw[(2 * t4) * 16 + kk], p1 = pw[(2 * t4 + 1) * 16 + kk];
            while (bits) {
              const int j = __ffs(bits) - 1;
              bits &= bits - 1u;
              const ushort4 hv = payload(1, pay_row(vax, kw0 + kk, fv, 4 * g4 + j));
              const float x[4] = {__half2float(__ushort_as_half(hv.x)),
                                  __half2float(__ushort_as_half(hv.y)),
                                  __half2float(__ushort_as_half(hv.z)),
                                  __half2float(__ushort_as_half(hv.w))};
#pragma unroll
              for (int jj = 0; jj < 4; ++jj) {
                if (jj != j) continue;  // register-resident oT: compile-time indices
#pragma unroll
                for (int d = 0; d < 4; ++d) {
                  oT[2 * jj + (d >> 1)][(d & 1) * 2 + 0] += p0 * x[d];
                  oT[2 * jj + (d >> 1)][(d & 1) * 2 + 1] += p1 * x[d];
                }
              }
            }
          }
          __syncwarp();
        }
        release(k, stage);
      }
    } else {
      release(k, stage);
    }
  }
  // every consumer is past its last read of the ring (and no bulk copy is in
  // flight: each issued tile was consumed) -> reuse the ring for the merge
  __syncthreads();
  {
    float* mo = reinterpret_cast<float*>(ring);  // [warp][row][130]
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int row = t4 * 2 + (e & 1);
        const int dim = 4 * (4 * g4 + (mt >> 1)) + 2 * (mt & 1) + (e >> 1);
        mo[((size_t)warp * 8 + row) * 130 + dim] = oT[mt][e];
      }
    }
    if (t4 == 0) {
      mo[((size_t)warp * 8 + g4) * 130 + 128] = m_run;
      mo[((size_t)warp * 8 + g4) * 130 + 129] = l_run;
    }
  }
  __syncthreads();
  // ---- merge the consumers' (m, l, O) and write
  const float* mo = reinterpret_cast<const float*>(ring);
  for (int i = tid; i < 8 * 128; i += kMThreads) {
    const int r = i >> 7, d = i & 127;
    if (r >= p.nrows) continue;
    float M = -INFINITY;
#pragma unroll
    for (int ww = 0; ww < kMConsumers; ++ww) M = fmaxf(M, mo[((size_t)ww * 8 + r) * 130 + 128]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int ww = 0; ww < kMConsumers; ++ww) {
        const float* st = mo + ((size_t)ww * 8 + r) * 130;
        if (st[128] != -INFINITY) {
          const float f = exp2f(st[128] - M);
          L += st[129] * f;
          O += st[d] * f;
        }
      }
    }
    const int gi = r / (int)p.Tq, qi = r - gi * (int)p.Tq;
    const int64_t hq = hkv * p.g + gi;
    if (p.splits == 1) {
      // (fast divide: an IEEE '/' here is a subroutine call, which makes ptxas keep
      // the global-memory descriptor out of the uniform registers kernel-wide)
      p.out[((b * p.Hq + hq) * p.Tq + qi) * 128 + d] = __fdividef(O, L);
    } else {
      const int64_t idx = (bh * p.nrows + r) * p.splits + blockIdx.x;
      p.part_o[idx * 128 + d] = O;
      if (d == 0) {
        p.part_ml[2 * idx] = M;
        p.part_ml[2 * idx + 1] = L;
      }
    }
  }
}


size_t prefill_tc_workspace(const hqmq_attention_args* a);
bool prefill_tc_applicable(const hqmq_attention_args* a);
int launch_prefill_tc(const hqmq_attention_args* a, cudaStream_t st);
// attention_cluster.cu: the K/V CTA-pair decode kernel
bool pair_applicable(int64_t bhkv, int64_t head_dim, int64_t nrows, int64_t tkv, int S, int w, int br,
                     bool flags, const void* t16k, const void* t16v);
size_t pair_workspace(int64_t bhkv, int64_t nrows, int64_t tkv);
int launch_pair_attention(AttParams p, int64_t max_tkv, cudaStream_t st);
static bool al16(const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; }
static bool pair_ok(const hqmq_attention_args* a) {
#ifdef HQMQ_DISABLE_PAIR
  return false;
#endif
  const int64_t nrows = a->q_heads / a->kv_heads * a->q_tokens;
  return !a->precise &&
         pair_applicable(a->batch * a->kv_heads, a->head_dim, nrows, a->kv_tokens, a->codebook_size, a->index_bits,
                         a->radius_bits, a->k.flag_words || a->v.flag_words, a->k.joint_f16,
                         a->v.joint_f16) &&
         al16(a->k.index_words) && al16(a->k.radius_words) && al16(a->k.scales) &&
         al16(a->v.index_words) && al16(a->v.radius_words) && al16(a->v.scales);
}

namespace {

struct AttPlan {
  int splits;
  int64_t keys_per_split;
  int row_groups;
  size_t ws;
};

bool plan_att(const hqmq_attention_args* a, AttPlan& pl) {
  if (!a || a->batch < 1 || a->q_heads < 1 || a->kv_heads < 1 || a->q_tokens < 1 ||
      a->kv_tokens < 1 || a->head_dim < 1)
    return false;
  if (a->q_heads % a->kv_heads) return false;
  if (a->head_dim % 4 || a->head_dim > 4 * kMaxC) return false;
  if (a->causal && a->q_tokens > a->kv_tokens) return false;
  const int64_t g = a->q_heads / a->kv_heads;
  const int64_t nrows = g * a->q_tokens;
  pl.row_groups = (int)ceil_div(nrows, kRows);
  const int64_t ctas = a->batch * a->kv_heads * pl.row_groups;
  int splits = a->num_splits;
  if (splits <= 0) {
    // Per-SM load model: a split costs its 128-key tiles plus ~3 tiles of
    // prologue (table staging, ring fill) and the busiest of the 148 SMs
    // runs ceil(ctas*splits/148) CTAs; pick the cheapest split count.
    int64_t best = INT64_MAX;
    splits = 1;
    const int64_t max_s = std::max<int64_t>(1, std::min<int64_t>(64, ceil_div(a->kv_tokens, 256)));
    for (int64_t s = 1; s <= max_s; ++s) {
      const int64_t tiles = ceil_div(ceil_div(a->kv_tokens, s), 128);
      // waves of 2 CTAs per SM (296 slots), one tile of per-CTA overhead
      // (measured at C4: 8 splits 0.611 ms vs the old model's 4 at 0.617)
      const int64_t cost = ceil_div(ctas * s, 2 * 148) * (tiles + 1);
      if (cost < best) {
        best = cost;
        splits = (int)s;
      }
    }
  }
  pl.keys_per_split = ceil_div(ceil_div(a->kv_tokens, splits), 64) * 64;
  pl.splits = (int)ceil_div(a->kv_tokens, pl.keys_per_split);
  const int64_t parts = a->batch * a->kv_heads * nrows * pl.splits;
  const size_t elt = a->precise == 2 ? sizeof(double) : sizeof(float);
  pl.ws = pl.splits > 1 ? (size_t)parts * (a->head_dim + 2) * elt + 256 : 0;
  if (prefill_tc_applicable(a)) pl.ws = std::max(pl.ws, prefill_tc_workspace(a));
  if (pair_ok(a)) pl.ws = std::max(pl.ws, pair_workspace(a->batch * a->kv_heads, nrows, a->kv_tokens));
  return true;
}

}  // namespace
}  // namespace hqmq

namespace hqmq {
namespace {
enum AttKind { kAttF64, kAttPrefillTc, kAttPair, kAttMma, kAttMmaMed3x, kAttSplitSmem, kAttSplit };
struct AttChoice {
  AttKind kind;
  void (*mk)(AttParams);
  size_t msmem;
};
const char* att_kind_name(AttKind k) {
  switch (k) {
    case kAttF64: return "attention_f64_kernel";
    case kAttPrefillTc: return "prefill_tc (tcgen05 flash attention)";
    case kAttPair: return "attention_pair_kernel (K/V CTA pair)";
    case kAttMma: return "attention_mma_kernel";
    case kAttMmaMed3x: return "attention_mma_kernel<Med3x>";
    case kAttSplitSmem: return "attention_split_kernel<smem>";
    default: return "attention_split_kernel";
  }
}
// Which kernel hqmq_attention_decode runs for `a` (the plan already checked).
AttChoice choose_att(const hqmq_attention_args* a, const AttPlan& pl) {
  AttChoice ch{kAttSplit, nullptr, 0};
  if (a->precise == 2) {
    ch.kind = kAttF64;
    return ch;
  }
  const int64_t nrows = a->q_heads / a->kv_heads * a->q_tokens;
  const size_t tab_bytes = 2 * (size_t)kGroupOrder * a->codebook_size * sizeof(float4);
  // Med3x caches take the same tensor-core kernel (kFlags): both tensors must
  // carry the flag bitmap, token offsets and payload rows
  const bool flags = a->k.flag_words && a->v.flag_words && a->k.token_offsets &&
                     a->v.token_offsets && a->k.payloads && a->v.payloads;
  const bool flags_mixed = (a->k.flag_words != nullptr) != (a->v.flag_words != nullptr);
  const size_t msmem = mma_smem_bytes(a->codebook_size, a->index_bits, a->radius_bits, flags);
  const bool mma_path = a->head_dim == 128 && !flags_mixed &&
                        (flags || (!a->k.flag_words && !a->v.flag_words)) &&
                        nrows <= 8 && a->kv_tokens % 8 == 0 && pl.keys_per_split % 64 == 0 &&
                        msmem <= kMaxDynSmem && al16(a->k.index_words) && al16(a->k.radius_words) &&
                        al16(a->k.scales) && al16(a->v.index_words) && al16(a->v.radius_words) &&
                        al16(a->v.scales) && !a->precise &&
                        (!flags || (al16(a->k.flag_words) && al16(a->k.token_offsets) &&
                                    al16(a->v.flag_words) && al16(a->v.token_offsets)));
  // (index_bits, radius_bits) instances of the tensor-core kernel
  void (*mk)(AttParams) = nullptr;
  const int wb = a->index_bits * 16 + a->radius_bits;
  if (flags) {
    switch (wb) {
      case 9 * 16 + 4: mk = attention_mma_kernel<9, 4, false, true>; break;
      case 11 * 16 + 4: mk = attention_mma_kernel<11, 4, false, true>; break;
      case 11 * 16 + 6: mk = attention_mma_kernel<11, 6, false, true>; break;  // C3 (Qwen)
      case 13 * 16 + 4: mk = attention_mma_kernel<13, 4, false, true>; break;
      default: break;
    }
  } else switch (wb) {
    case 9 * 16 + 4: mk = attention_mma_kernel<9, 4>; break;    // S = 16..21, b_r 4
    case 10 * 16 + 4: mk = attention_mma_kernel<10, 4>; break;
    case 11 * 16 + 4: mk = attention_mma_kernel<11, 4>; break;  // S = 43..85 (S=64), b_r 4
    case 12 * 16 + 4: mk = attention_mma_kernel<12, 4>; break;
    case 13 * 16 + 4: mk = attention_mma_kernel<13, 4>; break;  // S = 171..341 (S=256)
    case 11 * 16 + 6: mk = attention_mma_kernel<11, 6>; break;  // Qwen config b_r 6
    case 11 * 16 + 3: mk = attention_mma_kernel<11, 3>; break;
    case 12 * 16 + 3: mk = attention_mma_kernel<12, 3>; break;
    default: break;
  }
  if (prefill_tc_applicable(a)) {
    ch.kind = kAttPrefillTc;
  } else if (pair_ok(a)) {
    ch.kind = kAttPair;
  } else if (mma_path && mk) {
    ch.kind = flags ? kAttMmaMed3x : kAttMma;
    ch.mk = mk;
    ch.msmem = msmem;
  } else {
    ch.kind = tab_bytes <= 160 * 1024 ? kAttSplitSmem : kAttSplit;
  }
  return ch;
}
}  // namespace
}  // namespace hqmq

extern "C" {

size_t hqmq_attention_workspace_bytes(const hqmq_attention_args* a) {
  hqmq::AttPlan pl;
  if (!hqmq::plan_att(a, pl)) return 0;
  return pl.ws;
}

const char* hqmq_attention_kernel_name(const hqmq_attention_args* a) {
  hqmq::AttPlan pl;
  if (!hqmq::plan_att(a, pl)) return "invalid";
  return hqmq::att_kind_name(hqmq::choose_att(a, pl).kind);
}

int hqmq_attention_decode(const hqmq_attention_args* a, void* stream) {
  using namespace hqmq;
  AttPlan pl;
  if (!plan_att(a, pl)) return HQMQ_ERR_INVALID_ARGUMENT;
  if (a->workspace_bytes < pl.ws) return HQMQ_ERR_WORKSPACE;
  if (a->codebook_size < 1 || a->radius_bits < 1 || a->radius_bits > 8 || a->index_bits < 1 ||
      a->index_bits > 32)
    return HQMQ_ERR_INVALID_ARGUMENT;
  if (a->batch * a->kv_heads >= 65536 || pl.row_groups >= 65536) return HQMQ_ERR_UNSUPPORTED;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  AttParams p;
  p.B = a->batch; p.Hq = a->q_heads; p.Hkv = a->kv_heads; p.Tq = a->q_tokens;
  p.Tkv = a->kv_tokens; p.D = a->head_dim;
  p.C = (int)(a->head_dim / 4); p.S = a->codebook_size; p.br = a->radius_bits; p.w = a->index_bits;
  p.g = (int)(a->q_heads / a->kv_heads); p.causal = a->causal;
  p.scale_log2 = (float)(a->scale * 1.4426950408889634);
  p.o_scale = 1.0f;
  p.splits = pl.splits; p.keys_per_split = pl.keys_per_split;
  p.nrows = (int)(p.g * a->q_tokens);
  p.kv_lens = nullptr; p.block_table = nullptr; p.max_pages = 0;
  p.q = a->q;
  auto view = [](const hqmq_packed_view& v) {
    AttView o;
    o.scales = v.scales; o.idxw = v.index_words; o.radw = v.radius_words; o.flagw = v.flag_words;
    o.payloads = v.payloads; o.tokoff = v.token_offsets;
    o.table = reinterpret_cast<const float4*>(v.joint_f32);
    o.table16 = reinterpret_cast<const uint2*>(v.joint_f16);
    o.table64 = v.joint_f64;
    return o;
  };
  p.k = view(a->k);
  p.v = view(a->v);
  p.out = a->out;
  if (a->precise == 2) {  // fp64 contract (attention.py:137-145 default dtype)
    if (!a->k.joint_f64 || !a->v.joint_f64) return HQMQ_ERR_INVALID_ARGUMENT;
    AttParams64 p64;
    p64.q = reinterpret_cast<const double*>(a->q);
    p64.out = reinterpret_cast<double*>(a->out);
    double* ws64 = reinterpret_cast<double*>(a->workspace);
    const int64_t parts64 = a->batch * a->kv_heads * p.nrows * pl.splits;
    p64.part_o = ws64;
    p64.part_ml = ws64 ? ws64 + parts64 * a->head_dim : nullptr;
    p64.scale = a->scale;
    const size_t sm64 = f64_smem_bytes();
    cudaFuncSetAttribute(attention_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm64);
    const dim3 g64((unsigned)pl.splits, (unsigned)(a->batch * a->kv_heads), (unsigned)pl.row_groups);
    attention_f64_kernel<<<g64, kAttThreads, sm64, st>>>(p, p64);
    int rc = check_launch();
    if (rc != HQMQ_OK || pl.splits == 1) return rc;
    combine_f64_kernel<<<dim3((unsigned)(a->batch * a->kv_heads), (unsigned)p.nrows), 128, 0, st>>>(p, p64);
    return check_launch();
  }
  float* ws = reinterpret_cast<float*>(a->workspace);
  const int64_t parts = a->batch * a->kv_heads * p.nrows * pl.splits;
  p.part_o = ws;
  p.part_ml = ws ? ws + parts * a->head_dim : nullptr;
  const dim3 grid((unsigned)pl.splits, (unsigned)(a->batch * a->kv_heads), (unsigned)pl.row_groups);
  const AttChoice ch = choose_att(a, pl);
  if (ch.kind == kAttPrefillTc) return launch_prefill_tc(a, st);
  if (ch.kind == kAttPair) {
    p.part_o = ws;
    return launch_pair_attention(p, a->kv_tokens, st);
  }
  if (ch.kind == kAttMma || ch.kind == kAttMmaMed3x) {
    cudaFuncSetAttribute(ch.mk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDynSmem);
    ch.mk<<<dim3((unsigned)pl.splits, (unsigned)(a->batch * a->kv_heads)), kMThreads, ch.msmem, st>>>(p);
  } else if (ch.kind == kAttSplitSmem) {
    const size_t tab_bytes = 2 * (size_t)kGroupOrder * a->codebook_size * sizeof(float4);
    cudaFuncSetAttribute(attention_split_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         160 * 1024);
    attention_split_kernel<true><<<grid, kAttThreads, tab_bytes, st>>>(p);
  } else {
    attention_split_kernel<false><<<grid, kAttThreads, 0, st>>>(p);
  }
  int rc = check_launch();
  if (rc != HQMQ_OK) return rc;
  if (pl.splits > 1) {
    combine_kernel<<<dim3((unsigned)(a->batch * a->kv_heads), (unsigned)p.nrows), 128, 0, st>>>(p);
    rc = check_launch();
  }
  return rc;
}

namespace {
struct PagedPlan {
  int splits;
  int64_t keys_per_split;
  size_t ws;
};
bool paged_pair_ok(const hqmq_paged_attention_args* a) {
#ifdef HQMQ_DISABLE_PAIR
  return false;
#endif
  return hqmq::pair_applicable(a->batch * a->kv_heads, a->head_dim, a->q_heads / a->kv_heads, a->max_kv_tokens, a->codebook_size,
                         a->index_bits, a->radius_bits, a->k.flag_pages || a->v.flag_pages,
                         a->k.joint_f16, a->v.joint_f16);
}
bool plan_paged(const hqmq_paged_attention_args* a, PagedPlan& pl) {
  using namespace hqmq;
  if (!a || a->batch < 1 || a->q_heads < 1 || a->kv_heads < 1 || a->head_dim != 128) return false;
  if (a->q_heads % a->kv_heads || a->q_heads / a->kv_heads > 8) return false;
  if (a->page_tokens != kMT || a->max_pages < 1 || a->max_kv_tokens < 1) return false;
  if ((int64_t)a->max_kv_tokens > (int64_t)a->max_pages * kMT) return false;
  const int64_t ctas = a->batch * a->kv_heads;
  int splits = a->num_splits;
  if (splits <= 0) {  // same per-SM load model as the contiguous path
    int64_t best = INT64_MAX;
    splits = 1;
    const int64_t max_s = std::max<int64_t>(1, std::min<int64_t>(64, ceil_div(a->max_kv_tokens, 256)));
    for (int64_t s = 1; s <= max_s; ++s) {
      const int64_t tiles = ceil_div(ceil_div(a->max_kv_tokens, s), kMT);
      const int64_t cost = ceil_div(ctas * s, 2 * 148) * (tiles + 1);
      if (cost < best) {
        best = cost;
        splits = (int)s;
      }
    }
  }
  pl.keys_per_split = ceil_div(ceil_div(a->max_kv_tokens, splits), kMT) * kMT;
  pl.splits = (int)ceil_div(a->max_kv_tokens, pl.keys_per_split);
  const int64_t nrows = a->q_heads / a->kv_heads;
  pl.ws = pl.splits > 1 ? (size_t)ctas * nrows * pl.splits * (128 + 2) * sizeof(float) + 256 : 0;
  if (paged_pair_ok(a)) pl.ws = std::max(pl.ws, pair_workspace(ctas, nrows, a->max_kv_tokens));
  return true;
}
}  // namespace

size_t hqmq_paged_attention_workspace_bytes(const hqmq_paged_attention_args* a) {
  PagedPlan pl;
  return plan_paged(a, pl) ? pl.ws : 0;
}

int hqmq_attention_decode_paged(const hqmq_paged_attention_args* a, void* stream) {
  using namespace hqmq;
  PagedPlan pl;
  if (!plan_paged(a, pl)) return HQMQ_ERR_INVALID_ARGUMENT;
  if (a->workspace_bytes < pl.ws) return HQMQ_ERR_WORKSPACE;
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (!al16(a->k.index_pages) || !al16(a->k.radius_pages) || !al16(a->k.scale_pages) ||
      !al16(a->v.index_pages) || !al16(a->v.radius_pages) || !al16(a->v.scale_pages))
    return HQMQ_ERR_INVALID_ARGUMENT;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  AttParams p;
  p.B = a->batch; p.Hq = a->q_heads; p.Hkv = a->kv_heads; p.Tq = 1; p.Tkv = a->max_kv_tokens;
  p.D = 128; p.C = 32; p.S = a->codebook_size; p.br = a->radius_bits; p.w = a->index_bits;
  p.g = (int)(a->q_heads / a->kv_heads); p.causal = 1;
  p.scale_log2 = (float)(a->scale * 1.4426950408889634);
  p.o_scale = 1.0f;
  p.splits = pl.splits; p.keys_per_split = pl.keys_per_split;
  p.nrows = p.g;
  p.q = a->q;
  auto view = [](const hqmq_paged_view& v) {
    AttView o;
    o.scales = v.scale_pages; o.idxw = v.index_pages; o.radw = v.radius_pages;
    // Med3x pages: flag words, and the payload row of each token's first
    // flagged chunk in the aux (token offset) slot
    o.flagw = v.flag_pages; o.payloads = v.payloads; o.tokoff = v.payoff_pages;
    o.table = reinterpret_cast<const float4*>(v.joint_f32);
    o.table16 = reinterpret_cast<const uint2*>(v.joint_f16);
    o.table64 = nullptr;
    return o;
  };
  p.k = view(a->k);
  p.v = view(a->v);
  p.out = a->out;
  float* ws = reinterpret_cast<float*>(a->workspace);
  const int64_t parts = a->batch * a->kv_heads * p.nrows * pl.splits;
  p.part_o = ws;
  p.part_ml = ws ? ws + parts * 128 : nullptr;
  p.kv_lens = a->kv_lens; p.block_table = a->block_table; p.max_pages = a->max_pages;
  if (paged_pair_ok(a)) return launch_pair_attention(p, a->max_kv_tokens, st);
  void (*mk)(AttParams) = nullptr;
  const bool flags = a->k.flag_pages != nullptr;
  if (flags != (a->v.flag_pages != nullptr)) return HQMQ_ERR_INVALID_ARGUMENT;
  if (flags && (!a->k.payoff_pages || !a->v.payoff_pages || !a->k.payloads || !a->v.payloads ||
                !al16(a->k.flag_pages) || !al16(a->v.flag_pages) || !al16(a->k.payoff_pages) ||
                !al16(a->v.payoff_pages)))
    return HQMQ_ERR_INVALID_ARGUMENT;
  switch (a->index_bits * 16 + a->radius_bits + (flags ? 1024 : 0)) {
    case 9 * 16 + 4: mk = attention_mma_kernel<9, 4, true>; break;
    case 11 * 16 + 4: mk = attention_mma_kernel<11, 4, true>; break;
    case 13 * 16 + 4: mk = attention_mma_kernel<13, 4, true>; break;
    case 11 * 16 + 6: mk = attention_mma_kernel<11, 6, true>; break;
    case 1024 + 9 * 16 + 4: mk = attention_mma_kernel<9, 4, true, true>; break;
    case 1024 + 11 * 16 + 4: mk = attention_mma_kernel<11, 4, true, true>; break;
    case 1024 + 13 * 16 + 4: mk = attention_mma_kernel<13, 4, true, true>; break;
    case 1024 + 11 * 16 + 6: mk = attention_mma_kernel<11, 6, true, true>; break;
    default: return HQMQ_ERR_UNSUPPORTED;
  }
  const size_t msmem = mma_smem_bytes(a->codebook_size, a->index_bits, a->radius_bits, flags);
  if (msmem > kMaxDynSmem) return HQMQ_ERR_UNSUPPORTED;
  cudaFuncSetAttribute(mk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxDynSmem);
  mk<<<dim3((unsigned)pl.splits, (unsigned)(a->batch * a->kv_heads)), kMThreads, msmem, st>>>(p);
  int rc = check_launch();
  if (rc != HQMQ_OK) return rc;
  if (pl.splits > 1) {
    combine_kernel<<<dim3((unsigned)(a->batch * a->kv_heads), (unsigned)p.nrows), 128, 0, st>>>(p);
    rc = check_launch();
  }
  return rc;
}

}  // extern "C"
