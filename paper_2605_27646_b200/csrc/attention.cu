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
#include <cfloat>
#include <cmath>

#include "common.cuh"

namespace hqmq {

constexpr int kAttThreads = 128;
constexpr int kKT = 32;          // keys per tile
constexpr int kRows = 4;         // query rows per CTA (one warp each)
constexpr int kMaxC = 32;        // head_dim <= 128
constexpr int kKStride = 4 * kMaxC + 4;  // padded smem row (floats)

struct AttView {
  const uint16_t* scales;
  const uint32_t* idxw;
  const uint32_t* radw;
  const uint32_t* flagw;
  const uint16_t* payloads;
  const uint32_t* tokoff;
  const float4* table;  // [Hkv][24S]
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
};

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
  const int64_t b = bh / p.Hkv, hkv = bh % p.Hkv;
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
  const int64_t b = bh / p.Hkv, hkv = bh % p.Hkv;
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
    o[d] = acc / L;
  }
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
    const int64_t target = 148 * 8;
    splits = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(target, ctas),
                                                           ceil_div(a->kv_tokens, 256)));
  }
  pl.keys_per_split = ceil_div(ceil_div(a->kv_tokens, splits), kKT) * kKT;
  pl.splits = (int)ceil_div(a->kv_tokens, pl.keys_per_split);
  const int64_t parts = a->batch * a->kv_heads * nrows * pl.splits;
  pl.ws = pl.splits > 1 ? (size_t)parts * (a->head_dim + 2) * sizeof(float) + 256 : 0;
  return true;
}

}  // namespace
}  // namespace hqmq

extern "C" {

size_t hqmq_attention_workspace_bytes(const hqmq_attention_args* a) {
  hqmq::AttPlan pl;
  if (!hqmq::plan_att(a, pl)) return 0;
  return pl.ws;
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
  p.splits = pl.splits; p.keys_per_split = pl.keys_per_split;
  p.nrows = (int)(p.g * a->q_tokens);
  p.q = a->q;
  auto view = [](const hqmq_packed_view& v) {
    AttView o;
    o.scales = v.scales; o.idxw = v.index_words; o.radw = v.radius_words; o.flagw = v.flag_words;
    o.payloads = v.payloads; o.tokoff = v.token_offsets;
    o.table = reinterpret_cast<const float4*>(v.joint_f32);
    return o;
  };
  p.k = view(a->k);
  p.v = view(a->v);
  p.out = a->out;
  float* ws = reinterpret_cast<float*>(a->workspace);
  const int64_t parts = a->batch * a->kv_heads * p.nrows * pl.splits;
  p.part_o = ws;
  p.part_ml = ws ? ws + parts * a->head_dim : nullptr;
  const size_t tab_bytes = 2 * (size_t)kGroupOrder * a->codebook_size * sizeof(float4);
  const dim3 grid((unsigned)pl.splits, (unsigned)(a->batch * a->kv_heads), (unsigned)pl.row_groups);
  if (tab_bytes <= 160 * 1024) {
    static thread_local bool set = false;
    if (!set) {
      cudaFuncSetAttribute(attention_split_kernel<true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024);
      set = true;
    }
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

}  // extern "C"
