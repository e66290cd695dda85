// HQMQ decode for sm_100a (HBM-bound) plus the section pack / unpack / token
// offset / index validation helpers.
//
// Reference path replaced: codec.decode_token_range (codec.py:290-328),
// codec.decode_tensor (codec.py:331-336), radius.dequantize_radii
// (radius.py:50-54) and the kvpack stream codecs (kvpack.py:66-87,264-287).
//
// decode_kernel: one CTA column per (batch, head) row; the head's joint table
// (24*S codewords, fp32 or fp64) is staged once in shared memory and the CTA
// then streams its slice of the row: per chunk it reads w + b_r bits of the
// packed streams (funnel shift across 32-bit words) and the token's fp16
// scale, gathers the codeword from smem and writes the 4 reconstructed
// elements.  Flagged chunks come from the fp16 payload rows, addressed through
// the per-token coded offsets.  The model shapes take the TMA-ring kernels:
// decode_fast_kernel (no extraction: token-aligned streams, two tokens per
// warp instruction) and decode_flag_tma_kernel (Med3x: a 64-token tile's
// compact code runs, flag words, offsets, scales and payload rows per ring
// stage, a chunk quad per lane); decode_f64_kernel is the bit-exact fp64 path;
// expand_kernel / paged_append_kernel serve the paged cache.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdio>
#include <type_traits>

#include "common.cuh"

namespace hqmq {

constexpr int kDecThreads = 256;
constexpr int kDecR = 4;
constexpr size_t kDecSmemLimit = 100 * 1024;

template <typename OutT>
struct Out;
template <>
struct Out<float> {
  static __device__ __forceinline__ float cvt(float v) { return v; }
};
template <>
struct Out<__half> {
  static __device__ __forceinline__ __half cvt(float v) { return __float2half_rn(v); }
};
template <>
struct Out<__nv_bfloat16> {
  static __device__ __forceinline__ __nv_bfloat16 cvt(float v) { return __float2bfloat16_rn(v); }
};

// r * codeword (fp16 table entry) rounded ONCE to fp16: the product in fp32
// (packed), then one RN conversion -- the fp16 output is fp16 of the fp32
// decode, not a double rounding through an fp16 radius
__device__ __forceinline__ uint2 mul_round_f16(float r, uint2 cw) {
  const float2 c01 = __half22float2(*reinterpret_cast<const __half2*>(&cw.x));
  const float2 c23 = __half22float2(*reinterpret_cast<const __half2*>(&cw.y));
  const float2 rr = make_float2(r, r);
  const float2 p01 = __fmul2_rn(rr, c01), p23 = __fmul2_rn(rr, c23);
  const __half2 h01 = __floats2half2_rn(p01.x, p01.y), h23 = __floats2half2_rn(p23.x, p23.y);
  return make_uint2(*reinterpret_cast<const uint32_t*>(&h01), *reinterpret_cast<const uint32_t*>(&h23));
}

struct DecParams {
  int64_t B, H, T, D;
  int C, S, br, w;
  int64_t t0, nt;  // token range start, count
  int aligned4;
  const uint16_t* scales;
  const uint32_t* idxw;
  const uint32_t* radw;
  const uint32_t* flagw;
  const uint16_t* payloads;
  const uint32_t* tokoff;
  const void* table;  // float4 [H][24S] or double [H][24S][4]
  const uint2* table16;  // optional fp16 [H][24S] (16-bit outputs)
  void* out;
  uint32_t* err;
  // fp16 output straight into UMMA tile layouts (prefill; 0 = row-major):
  // tiles of 2^tile_log2 keys, K-major (tile_mn 0) or MN-major (1), ntk per row
  int tile_log2 = 0, tile_mn = 0;
  int64_t tile_ntk = 0;
};

// 16-byte output unit (row-relative token tr, 8-dim group dg) in the tile layout
__device__ __forceinline__ int64_t tile_unit(const DecParams& p, int64_t row, int64_t tr, int dg) {
  const int kt = 1 << p.tile_log2;
  const int64_t tix = tr >> p.tile_log2;
  const int key = (int)(tr & (kt - 1));
  const int o = p.tile_mn ? dg * kt + (key >> 3) * 8 + (key & 7) : (key >> 3) * 128 + dg * 8 + (key & 7);
  return (row * p.tile_ntk + tix) * (int64_t)(kt * 16) + o;
}

// Coded-stream position of chunk (tok, c) and whether it is flagged.
__device__ __forceinline__ uint64_t coded_pos(const DecParams& p, int64_t tok, int c, bool& flagged) {
  const uint64_t g = (uint64_t)tok * p.C + c;
  if (!p.flagw) {
    flagged = false;
    return g;
  }
  flagged = (__ldg(p.flagw + (g >> 5)) >> (g & 31)) & 1u;
  // flagged chunks in [tok*C, g)
  uint64_t b = (uint64_t)tok * p.C;
  uint32_t nflag = 0;
  while (b < g) {
    const uint32_t word = __ldg(p.flagw + (b >> 5));
    const uint32_t sh = (uint32_t)(b & 31);
    const uint64_t take = min((uint64_t)(32 - sh), g - b);
    const uint32_t m = take == 32 ? 0xffffffffu : ((1u << take) - 1u);
    nflag += __popc((word >> sh) & m);
    b += take;
  }
  return (uint64_t)__ldg(p.tokoff + tok) + (uint64_t)(c - (int)nflag);
}

template <typename OutT, bool kSmem>
__global__ void __launch_bounds__(kDecThreads) decode_kernel(DecParams p) {
  extern __shared__ float4 tab_s[];
  const int64_t row = blockIdx.y;
  const int h = (int)((uint32_t)row % (uint32_t)p.H);  // (32-bit: no division subroutine)
  const int ncw = kGroupOrder * p.S;
  const float4* __restrict__ gtab = reinterpret_cast<const float4*>(p.table) + (int64_t)h * ncw;
  if (kSmem) {
    for (int i = threadIdx.x; i < ncw; i += kDecThreads) tab_s[i] = __ldg(gtab + i);
    __syncthreads();
  }
  const float4* tab = kSmem ? tab_s : gtab;
  const int C = p.C, w = p.w, br = p.br;
  const float rtop = 1.0f / (float)((1 << br) - 1);
  const int64_t nck = p.nt * C;  // chunks of this row in range
  const int64_t per_blk = ceil_div(ceil_div(nck, gridDim.x), (int64_t)C) * C;
  const int64_t beg = (int64_t)blockIdx.x * per_blk;
  const int64_t end = min(nck, beg + per_blk);
  OutT* __restrict__ out = reinterpret_cast<OutT*>(p.out);
  for (int64_t base = beg; base < end; base += kDecThreads * kDecR) {
#pragma unroll
    for (int j = 0; j < kDecR; ++j) {
      const int64_t ci = base + j * kDecThreads + threadIdx.x;
      if (ci >= end) continue;
      const int64_t tr = ci / C;
      const int c = (int)(ci - tr * C);
      const int64_t tok = row * p.T + p.t0 + tr;
      bool fl;
      const uint64_t pos = coded_pos(p, tok, c, fl);
      float v[4];
      if (!fl) {
        uint32_t idx = read_bits(p.idxw, pos * (uint64_t)w, w);
        const uint32_t q = read_bits(p.radw, pos * (uint64_t)br, br);
        if (idx >= (uint32_t)ncw) {
          atomicOr(p.err, HQMQ_DEVERR_INDEX_RANGE);
          idx = 0;
        }
        const float sig = __half2float(__ushort_as_half(__ldg(p.scales + tok)));
        const float rad = ((float)q * sig) * rtop;
        const float4 cw = tab[idx];
        v[0] = rad * cw.x; v[1] = rad * cw.y; v[2] = rad * cw.z; v[3] = rad * cw.w;
      } else {
        const uint64_t prow = (uint64_t)tok * C + c - pos;
        const ushort4 hv = __ldg(reinterpret_cast<const ushort4*>(p.payloads) + prow);
        v[0] = __half2float(__ushort_as_half(hv.x));
        v[1] = __half2float(__ushort_as_half(hv.y));
        v[2] = __half2float(__ushort_as_half(hv.z));
        v[3] = __half2float(__ushort_as_half(hv.w));
      }
      OutT* o = out + (row * p.nt + tr) * p.D + 4 * c;
      if (p.aligned4) {
        if constexpr (sizeof(OutT) == 4) {
          *reinterpret_cast<float4*>(o) = make_float4(v[0], v[1], v[2], v[3]);
        } else {
          OutT tmp[4] = {Out<OutT>::cvt(v[0]), Out<OutT>::cvt(v[1]), Out<OutT>::cvt(v[2]),
                         Out<OutT>::cvt(v[3])};
          *reinterpret_cast<uint2*>(o) = *reinterpret_cast<const uint2*>(tmp);
        }
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (4 * c + i < p.D) o[i] = Out<OutT>::cvt(v[i]);
      }
    }
  }
}

// ------------------------------------------------ TMA-pipelined fast path
// Token-aligned layout (head_dim 128, no extraction): token t's codes are the
// index_bits words [t*w, (t+1)*w) and radius_bits words [t*br, (t+1)*br).  A
// CTA owns one (batch, head) row slice; thread 0 streams 64-token tiles of the
// three sections into a kFDStages-deep shared-memory ring with 1-D bulk
// copies (cp.async.bulk, completion on an mbarrier) while all 8 warps decode
// the previous tiles (warp = token, lane = chunk) and write coalesced rows.
#ifndef HQMQ_FD_TOK
#define HQMQ_FD_TOK 128
#endif
#ifndef HQMQ_FD_STAGES
#define HQMQ_FD_STAGES 2
#endif
constexpr int kFDTok = HQMQ_FD_TOK;        // tokens per ring tile
constexpr int kFDStages = HQMQ_FD_STAGES;  // ring depth

struct FastDecodeGeom {
  uint32_t idx_off, rad_off, sc_off, stage_bytes;
};

__host__ __device__ inline FastDecodeGeom fd_geom(int w, int br) {
  FastDecodeGeom g;
  const uint32_t ib = kFDTok * w * 4 + 16, rb = kFDTok * br * 4 + 16, sb = kFDTok * 2;
  g.idx_off = 0;
  g.rad_off = (ib + 127) / 128 * 128;
  g.sc_off = g.rad_off + (rb + 127) / 128 * 128;
  g.stage_bytes = g.sc_off + (sb + 127) / 128 * 128;
  return g;
}

// One token of the fast path: lane = chunk.  W / BR compile-time (0 = read
// from p): the lane's bit offsets inside a token are then constants, and the
// token stride (W words of index codes, BR words of radius codes) folds into
// immediate load offsets when the caller unrolls over tokens.
template <typename OutT, int W, int BR, bool kTile = false>
__device__ __forceinline__ void decode_token_fast(const DecParams& p, const uint32_t* __restrict__ iw,
                                                  const uint32_t* __restrict__ rw,
                                                  const uint16_t* __restrict__ sc,
                                                  const float4* __restrict__ tab, int tt,
                                                  OutT* __restrict__ o, int lane, uint32_t ncw,
                                                  float rtop, bool& bad, int64_t row = 0,
                                                  int64_t tr = 0) {
  if constexpr (sizeof(OutT) == 2 && kTile)  // half a 16-byte unit: chunk `lane` of token tr
    o = reinterpret_cast<OutT*>(reinterpret_cast<uint4*>(p.out) + tile_unit(p, row, tr, lane >> 1)) +
        4 * (lane & 1);
  const int w = W ? W : p.w, br = BR ? BR : p.br;
  const uint32_t imask = w == 32 ? 0xffffffffu : ((1u << w) - 1u);
  const uint32_t rmask = (1u << br) - 1u;
  const uint32_t bi = (uint32_t)lane * w, bq = (uint32_t)lane * br;
  const uint32_t* wp = iw + tt * w + (bi >> 5);
  uint32_t idx = __funnelshift_r(wp[0], wp[1], bi & 31) & imask;
  const uint32_t* qp = rw + tt * br + (bq >> 5);
  uint32_t q;
  if ((BR != 0) && (32 % (BR ? BR : 1) == 0)) q = (qp[0] >> (bq & 31)) & rmask;
  else q = __funnelshift_r(qp[0], qp[1], bq & 31) & rmask;
  bad |= idx >= ncw;  // reported once per thread at the end (no branch here)
  idx = idx < ncw ? idx : 0u;
  const float rad = (float)q * (__half2float(__ushort_as_half(sc[tt])) * rtop);
  if constexpr (sizeof(OutT) == 4) {
    const float4 cw = tab[idx];
    *reinterpret_cast<float4*>(o) = make_float4(rad * cw.x, rad * cw.y, rad * cw.z, rad * cw.w);
  } else {
    // 16-bit outputs gather from the fp16 copy of the table (8-byte entries:
    // half the shared-memory wavefronts of the fp32 gather, the kernel's
    // bottleneck); the extra rounding is far below the output's own ulp.
    const uint2 cw = reinterpret_cast<const uint2*>(tab)[idx];
    const __half2 c01 = *reinterpret_cast<const __half2*>(&cw.x);
    const __half2 c23 = *reinterpret_cast<const __half2*>(&cw.y);
    uint2 ov;
    if constexpr (std::is_same<OutT, __half>::value) {
      ov = mul_round_f16(rad, cw);
    } else {
      const float2 f01 = __half22float2(c01), f23 = __half22float2(c23);
      const __nv_bfloat162 o01 = __floats2bfloat162_rn(rad * f01.x, rad * f01.y);
      const __nv_bfloat162 o23 = __floats2bfloat162_rn(rad * f23.x, rad * f23.y);
      ov = make_uint2(*reinterpret_cast<const uint32_t*>(&o01), *reinterpret_cast<const uint32_t*>(&o23));
    }
    *reinterpret_cast<uint2*>(o) = ov;
  }
}

// Two tokens per warp instruction (compile-time W / BR only): half-warp h
// takes token tt + h, lane l = lane & 15 decodes chunks 2l and 2l+1, so one
// pair of code loads feeds two chunks and the row store is 16 bytes per lane.
template <typename OutT, int W, int BR, bool kTile = false>
__device__ __forceinline__ void decode_token2_fast(const uint32_t* __restrict__ iw,
                                                   const uint32_t* __restrict__ rw,
                                                   const uint16_t* __restrict__ sc,
                                                   const void* __restrict__ tab, int tt,
                                                   OutT* __restrict__ orow, int lane, uint32_t ncw,
                                                   float rtop, bool& bad, const DecParams& p,
                                                   int64_t row, int64_t tr0) {
  constexpr uint32_t kIM = W == 32 ? 0xffffffffu : ((1u << W) - 1u);
  constexpr uint32_t kRM = (1u << BR) - 1u;
  const int t = tt + (lane >> 4);
  const uint32_t c0 = 2u * (uint32_t)(lane & 15);
  const uint32_t bi = c0 * W, bq = c0 * BR;
  const uint32_t* wp = iw + t * W + (bi >> 5);
  static_assert(2 * W <= 32 && 2 * BR <= 32, "two codes must fit one funnel-shifted word");
  const uint32_t ipair = __funnelshift_r(wp[0], wp[1], bi & 31);  // 2W <= 32 bits from bi
  uint32_t i0 = ipair & kIM;
  uint32_t i1 = (ipair >> W) & kIM;
  const uint32_t* qp = rw + t * BR + (bq >> 5);
  uint32_t qpair;
  if constexpr ((32 % (2 * BR)) == 0) qpair = qp[0] >> (bq & 31);
  else qpair = __funnelshift_r(qp[0], qp[1], bq & 31);
  const uint32_t q0 = qpair & kRM, q1 = (qpair >> BR) & kRM;
  bad |= (i0 >= ncw) | (i1 >= ncw);
  i0 = i0 < ncw ? i0 : 0u;
  i1 = i1 < ncw ? i1 : 0u;
  const float sg = __half2float(__ushort_as_half(sc[t])) * rtop;
  const float r0 = (float)q0 * sg, r1 = (float)q1 * sg;
  OutT* o = orow + t * 128 + 4 * c0;
  if constexpr (sizeof(OutT) == 2 && kTile)  // the unit (token, dims 8l..8l+7)
    o = reinterpret_cast<OutT*>(reinterpret_cast<uint4*>(p.out) + tile_unit(p, row, tr0 + t, lane & 15));
  if constexpr (sizeof(OutT) == 4) {
    const float4 a = reinterpret_cast<const float4*>(tab)[i0];
    const float4 b = reinterpret_cast<const float4*>(tab)[i1];
    reinterpret_cast<float4*>(o)[0] = make_float4(r0 * a.x, r0 * a.y, r0 * a.z, r0 * a.w);
    reinterpret_cast<float4*>(o)[1] = make_float4(r1 * b.x, r1 * b.y, r1 * b.z, r1 * b.w);
  } else {
    const uint2 a = reinterpret_cast<const uint2*>(tab)[i0];
    const uint2 b = reinterpret_cast<const uint2*>(tab)[i1];
    uint4 ov;
    if constexpr (std::is_same<OutT, __half>::value) {
      const uint2 x01 = mul_round_f16(r0, a), x23 = mul_round_f16(r1, b);
      ov = make_uint4(x01.x, x01.y, x23.x, x23.y);
    } else {
      const float2 a01 = __half22float2(*reinterpret_cast<const __half2*>(&a.x));
      const float2 a23 = __half22float2(*reinterpret_cast<const __half2*>(&a.y));
      const float2 b01 = __half22float2(*reinterpret_cast<const __half2*>(&b.x));
      const float2 b23 = __half22float2(*reinterpret_cast<const __half2*>(&b.y));
      const __nv_bfloat162 x0 = __floats2bfloat162_rn(r0 * a01.x, r0 * a01.y);
      const __nv_bfloat162 x1 = __floats2bfloat162_rn(r0 * a23.x, r0 * a23.y);
      const __nv_bfloat162 x2 = __floats2bfloat162_rn(r1 * b01.x, r1 * b01.y);
      const __nv_bfloat162 x3 = __floats2bfloat162_rn(r1 * b23.x, r1 * b23.y);
      ov = make_uint4(*reinterpret_cast<const uint32_t*>(&x0), *reinterpret_cast<const uint32_t*>(&x1),
                      *reinterpret_cast<const uint32_t*>(&x2), *reinterpret_cast<const uint32_t*>(&x3));
    }
    *reinterpret_cast<uint4*>(o) = ov;
  }
}

// Shared-memory table bytes: fp32 codewords for fp32 output, fp16 copies
// (8-byte entries) for 16-bit outputs; the TMA ring starts after them.
template <typename OutT>
__host__ __device__ inline size_t fd_table_bytes(int ncw) {
  const size_t b = (size_t)ncw * (sizeof(OutT) == 4 ? 16 : 8);
  return (b + 127) / 128 * 128;
}

template <typename OutT, int W, int BR, bool kTile = false>
__global__ void __launch_bounds__(256, 7) decode_fast_kernel(DecParams p) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t full[kFDStages];
  __shared__ __align__(8) uint64_t tab_bar;
  __shared__ unsigned int released[kFDStages];
  const int64_t row = blockIdx.y;
  const int h = (int)((uint32_t)row % (uint32_t)p.H);  // (32-bit: no division subroutine)
  const int ncw = kGroupOrder * p.S;
  const int w = W ? W : p.w, br = BR ? BR : p.br;
  const FastDecodeGeom g = fd_geom(w, br);
  float4* tab = reinterpret_cast<float4*>(dsm);
  unsigned char* ring = dsm + fd_table_bytes<OutT>(ncw);
  const float4* __restrict__ gtab = reinterpret_cast<const float4*>(p.table) + (int64_t)h * ncw;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntile = ceil_div(p.nt, kFDTok);
  const int64_t tok_base = row * p.T + p.t0;  // first token of the range in this row
  constexpr bool k16 = sizeof(OutT) == 2;
  const bool tab_tma = k16 && p.table16 != nullptr;

  auto issue = [&](int64_t tile, int stage) {
    const int64_t t = tok_base + tile * kFDTok;
    const int ntok = (int)min((int64_t)kFDTok, p.nt - tile * kFDTok);
    unsigned char* s = ring + (size_t)stage * g.stage_bytes;
    const uint32_t ib = ntok * w * 4, rb = ntok * br * 4, sb = ntok * 2;
    fence_proxy_async();
    mbar_arrive_expect_tx(&full[stage], ib + rb + sb);
    bulk_g2s(s + g.idx_off, p.idxw + t * w, ib, &full[stage]);
    bulk_g2s(s + g.rad_off, p.radw + t * br, rb, &full[stage]);
    bulk_g2s(s + g.sc_off, p.scales + t, sb, &full[stage]);
  };

  if (tid == 0) {
    for (int s = 0; s < kFDStages; ++s) {
      mbar_init(&full[s], 1);
      released[s] = 0u;
    }
    mbar_init(&tab_bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tid == 0) {
    if (tab_tma) {  // the fp16 table arrives by TMA beside the first tiles
      const uint32_t tb = (uint32_t)ncw * 8u;
      fence_proxy_async();
      mbar_arrive_expect_tx(&tab_bar, tb);
      bulk_g2s(tab, p.table16 + (int64_t)h * ncw, tb, &tab_bar);
    }
  }
  // the table load above reads constant codebook data; the code streams come
  // from an earlier kernel (the encode): wait for it (PDL), then let the next
  // kernel of the stream begin its own set-up
  pdl_wait();
  pdl_trigger();
  if (tid == 0) {
    int s = 0;
    for (int64_t tile = blockIdx.x; tile < ntile && s < kFDStages; tile += gridDim.x, ++s)
      issue(tile, s);
  }
  if constexpr (!k16) {
    for (int i = tid; i < ncw; i += 256) tab[i] = __ldg(gtab + i);
    __syncthreads();
  } else if (!tab_tma) {
    uint2* t16 = reinterpret_cast<uint2*>(tab);
    for (int i = tid; i < ncw; i += 256) {
      const float4 c = __ldg(gtab + i);
      const __half2 a = __floats2half2_rn(c.x, c.y), b = __floats2half2_rn(c.z, c.w);
      t16[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
    }
    __syncthreads();
  } else {
    mbar_wait(&tab_bar, 0u);
  }

  const float rtop = 1.0f / (float)((1 << br) - 1);
  OutT* __restrict__ out = reinterpret_cast<OutT*>(p.out);
  bool bad = false;
  int k = 0;
  for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x, ++k) {
    const int stage = k % kFDStages;
    mbar_wait(&full[stage], (uint32_t)((k / kFDStages) & 1));
    const unsigned char* s = ring + (size_t)stage * g.stage_bytes;
    const uint32_t* iw = reinterpret_cast<const uint32_t*>(s + g.idx_off);
    const uint32_t* rw = reinterpret_cast<const uint32_t*>(s + g.rad_off);
    const uint16_t* sc = reinterpret_cast<const uint16_t*>(s + g.sc_off);
    const int ntok = (int)min((int64_t)kFDTok, p.nt - tile * kFDTok);
    OutT* orow = out + (row * p.nt + tile * kFDTok) * 128 + 4 * lane;
    if (W != 0 && ntok == kFDTok) {
      // full tile, compile-time geometry: warp w decodes token pairs
      // (2w, 2w+1), (2w+16, 2w+17), ... (fully unrolled)
#pragma unroll
      for (int i = 0; i < kFDTok / 16; ++i)
        decode_token2_fast<OutT, W ? W : 1, BR ? BR : 1, kTile>(iw, rw, sc, tab, 2 * warp + 16 * i, orow - 4 * lane,
                                                        lane, (uint32_t)ncw, rtop, bad, p, row,
                                                        p.t0 + tile * kFDTok);
    } else if (ntok == kFDTok) {
      // full tile: warp w decodes tokens w, w+8, ..., w+56 (fully unrolled)
      const uint32_t* iww = iw + warp * w;
      const uint32_t* rww = rw + warp * br;
      const uint16_t* scw = sc + warp;
      OutT* ow = orow + warp * 128;
#pragma unroll
      for (int i = 0; i < kFDTok / 8; ++i)
        decode_token_fast<OutT, W, BR, kTile>(p, iww, rww, scw, tab, 8 * i, ow + 8 * i * 128, lane,
                                       (uint32_t)ncw, rtop, bad, row,
                                       p.t0 + tile * kFDTok + warp + 8 * i);
    } else {
      for (int tt = warp; tt < ntok; tt += 8)
        decode_token_fast<OutT, W, BR, kTile>(p, iw, rw, sc, tab, tt, orow + tt * 128, lane,
                                              (uint32_t)ncw, rtop, bad, row, p.t0 + tile * kFDTok + tt);
    }
    // release the stage without a block barrier: the last warp done with it
    // (acq_rel release count: every warp's reads precede the refill) issues
    // the tile kFDStages ahead into it
    __syncwarp();
    if (lane == 0) {
      if (stage_release(&released[stage]) == 7u) {
        released[stage] = 0u;
        const int64_t nxt = tile + (int64_t)kFDStages * gridDim.x;
        if (nxt < ntile) issue(nxt, stage);
      }
    }
  }
  if (bad) atomicOr(p.err, HQMQ_DEVERR_INDEX_RANGE);
}

// Med3x layout (head_dim 128, flag bitmap present): a token's 32 chunks own
// exactly flag word `tok`, and its coded chunks start at token_offsets[tok]
// in the index / radius streams.  Warp = token, lane = chunk; the warp's code
// reads hit one contiguous ~w-word span (L1), flagged lanes read their fp16
// payload row instead.  kU tokens per warp iteration for memory parallelism.
template <typename OutT>
__global__ void __launch_bounds__(256) decode_flag_kernel(DecParams p) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t tab_bar;
  constexpr int kU = 4;
  const int64_t row = blockIdx.y;
  const int h = (int)((uint32_t)row % (uint32_t)p.H);  // (32-bit: no division subroutine)
  const int ncw = kGroupOrder * p.S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr bool k16 = sizeof(OutT) == 2;
  float4* tab = reinterpret_cast<float4*>(dsm);
  const float4* __restrict__ gtab = reinterpret_cast<const float4*>(p.table) + (int64_t)h * ncw;
  const bool tab_tma = k16 && p.table16 != nullptr;
  if (tid == 0) {
    mbar_init(&tab_bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  if (tab_tma) {
    if (tid == 0) {
      const uint32_t tb = (uint32_t)ncw * 8u;
      fence_proxy_async();
      mbar_arrive_expect_tx(&tab_bar, tb);
      bulk_g2s(tab, p.table16 + (int64_t)h * ncw, tb, &tab_bar);
    }
    mbar_wait(&tab_bar, 0u);
  } else if constexpr (k16) {
    uint2* t16 = reinterpret_cast<uint2*>(tab);
    for (int i = tid; i < ncw; i += 256) {
      const float4 c = __ldg(gtab + i);
      const __half2 a = __floats2half2_rn(c.x, c.y), b = __floats2half2_rn(c.z, c.w);
      t16[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
    }
    __syncthreads();
  } else {
    for (int i = tid; i < ncw; i += 256) tab[i] = __ldg(gtab + i);
    __syncthreads();
  }
  const int w = p.w, br = p.br;
  const uint32_t imask = w == 32 ? 0xffffffffu : ((1u << w) - 1u);
  const uint32_t rmask = (1u << br) - 1u;
  const float rtop = 1.0f / (float)((1 << br) - 1);
  const uint32_t lt = (1u << lane) - 1u;
  OutT* __restrict__ out = reinterpret_cast<OutT*>(p.out);
  bool bad = false;
  const int64_t stride = (int64_t)gridDim.x * 8 * kU;
  for (int64_t t0 = ((int64_t)blockIdx.x * 8 + warp) * kU; t0 < p.nt; t0 += stride) {
    uint32_t fw[kU], off[kU];
    uint16_t scl[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t tt = min(t0 + u, p.nt - 1);
      const int64_t tok = row * p.T + p.t0 + tt;
      fw[u] = __ldg(p.flagw + tok);
      off[u] = __ldg(p.tokoff + tok);
      scl[u] = __ldg(p.scales + tok);
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int64_t tt = t0 + u;
      if (tt >= p.nt) break;
      const int64_t tok = row * p.T + p.t0 + tt;
      const bool fl = (fw[u] >> lane) & 1u;
      const uint64_t pos = (uint64_t)off[u] + __popc(~fw[u] & lt);
      float v[4];
      if (!fl) {
        uint32_t idx = read_bits(p.idxw, pos * (uint64_t)w, w) & imask;
        const uint32_t q = read_bits(p.radw, pos * (uint64_t)br, br) & rmask;
        bad |= idx >= (uint32_t)ncw;
        idx = idx < (uint32_t)ncw ? idx : 0u;
        const float rad = (float)q * (__half2float(__ushort_as_half(scl[u])) * rtop);
        if constexpr (k16) {
          const uint2 cw = reinterpret_cast<const uint2*>(tab)[idx];
          const float2 c01 = __half22float2(*reinterpret_cast<const __half2*>(&cw.x));
          const float2 c23 = __half22float2(*reinterpret_cast<const __half2*>(&cw.y));
          v[0] = rad * c01.x; v[1] = rad * c01.y; v[2] = rad * c23.x; v[3] = rad * c23.y;
        } else {
          const float4 cw = tab[idx];
          v[0] = rad * cw.x; v[1] = rad * cw.y; v[2] = rad * cw.z; v[3] = rad * cw.w;
        }
      } else {
        const uint64_t prow = (uint64_t)tok * 32 + lane - pos;
        const ushort4 hv = __ldg(reinterpret_cast<const ushort4*>(p.payloads) + prow);
        v[0] = __half2float(__ushort_as_half(hv.x));
        v[1] = __half2float(__ushort_as_half(hv.y));
        v[2] = __half2float(__ushort_as_half(hv.z));
        v[3] = __half2float(__ushort_as_half(hv.w));
      }
      OutT* o = out + (row * p.nt + tt) * 128 + 4 * lane;
      if constexpr (sizeof(OutT) == 4) {
        *reinterpret_cast<float4*>(o) = make_float4(v[0], v[1], v[2], v[3]);
      } else {
        OutT t4[4] = {Out<OutT>::cvt(v[0]), Out<OutT>::cvt(v[1]), Out<OutT>::cvt(v[2]),
                      Out<OutT>::cvt(v[3])};
        *reinterpret_cast<uint2*>(o) = *reinterpret_cast<const uint2*>(t4);
      }
    }
  }
  if (bad) atomicOr(p.err, HQMQ_DEVERR_INDEX_RANGE);
}

// Med3x layout through the TMA ring (head_dim 128): a 64-token tile's coded
// chunks are one contiguous run of the index / radius streams, [off[t0],
// off[t0+63] + coded(t0+63)), so the producer bulk-copies that run (16-byte
// aligned, with its base word recorded per stage) together with the tile's
// flag words, token offsets and scales; warps then decode like the fast path
// (warp = token, lane = chunk, coded position = token offset + ballot popc),
// flagged lanes reading their fp16 payload row from global.
#ifndef HQMQ_FL_STAGES
#define HQMQ_FL_STAGES 4
#endif
constexpr int kFlTok = 64;
constexpr int kFlStages = HQMQ_FL_STAGES;  // (sweep: tools/gpu_r4e.sh)

struct FlagGeom {
  uint32_t idx_off, rad_off, fl_off, to_off, sc_off, pay_off, stage_bytes;
};
// payload rows a stage can hold (the tile's outlier rows are one contiguous
// range of the payload section; a tile with more falls back to global loads)
constexpr int kFlPayRows = 256;
__host__ __device__ inline FlagGeom fl_geom(int w, int br) {
  auto up = [](uint32_t x) { return (x + 127u) / 128u * 128u; };
  FlagGeom g;
  uint32_t o = 0;
  g.idx_off = o; o += up((kFlTok * w + 8) * 4);
  g.rad_off = o; o += up((kFlTok * br + 8) * 4);
  g.fl_off = o; o += up(kFlTok * 4);
  g.to_off = o; o += up(kFlTok * 4);
  g.sc_off = o; o += up(kFlTok * 2);
  g.pay_off = o; o += up((kFlPayRows + 2) * 8);
  g.stage_bytes = o;
  return g;
}

// Med3x layout (head_dim 128): TMA ring of 64-token tiles holding the tile's
// compact index / radius words, flag words, coded offsets, scales and its
// outlier payload rows.  Two tokens per warp instruction (half-warp = token,
// lane = 2 chunks, 16-byte stores for fp16); a flagged chunk reads its fp16
// payload row from the stage.
template <typename OutT, int W = 0, int BR = 0>
__global__ void __launch_bounds__(256, 6) decode_flag_tma_kernel(DecParams p) {
  extern __shared__ __align__(128) unsigned char dsm[];
  __shared__ __align__(8) uint64_t full[kFlStages];
  __shared__ __align__(8) uint64_t tab_bar;
  __shared__ unsigned int released[kFlStages];
  // per stage: bit of the tile's first code in the staged index / radius
  // words, first staged payload row (64-bit), staged payload row count
  // (0 = the tile's rows are not staged: global loads)
  __shared__ uint32_t base_w[kFlStages][2];
  __shared__ unsigned long long pay_base[kFlStages];
  __shared__ uint32_t pay_n[kFlStages];
  const int64_t row = blockIdx.y;
  const int h = (int)((uint32_t)row % (uint32_t)p.H);  // (32-bit: no division subroutine)
  const int ncw = kGroupOrder * p.S;
  const int w = W ? W : p.w, br = BR ? BR : p.br;  // compile-time for the model configs
  const FlagGeom g = fl_geom(w, br);
  constexpr bool k16 = sizeof(OutT) == 2;
  float4* tab = reinterpret_cast<float4*>(dsm);
  const size_t tbytes = ((size_t)ncw * (k16 ? 8 : 16) + 127) / 128 * 128;
  unsigned char* ring = dsm + tbytes;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t ntile = ceil_div(p.nt, kFlTok);
  const int64_t tok_base = row * p.T + p.t0;
  const bool tab_tma = k16 && p.table16 != nullptr;

  auto issue = [&](int64_t tile, int stage) {
    const int64_t t = tok_base + tile * kFlTok;
    const int ntok = (int)min((int64_t)kFlTok, p.nt - tile * kFlTok);
    unsigned char* s = ring + (size_t)stage * g.stage_bytes;
    const uint64_t c0 = __ldg(p.tokoff + t);
    const uint64_t cl = __ldg(p.tokoff + t + ntok - 1);
    const uint32_t fl_last = __ldg(p.flagw + t + ntok - 1);
    const uint64_t c1 = cl + (uint64_t)__popc(~fl_last);
    const uint64_t iw0 = ((c0 * (uint64_t)w) >> 5) & ~3ull;
    const uint64_t iw1 = (((c1 * (uint64_t)w + 31) >> 5) + 3) & ~3ull;
    const uint64_t rw0 = ((c0 * (uint64_t)br) >> 5) & ~3ull;
    const uint64_t rw1 = (((c1 * (uint64_t)br + 31) >> 5) + 3) & ~3ull;
    base_w[stage][0] = (uint32_t)(c0 * (uint64_t)w - iw0 * 32u);   // c0's bit in the staged words
    base_w[stage][1] = (uint32_t)(c0 * (uint64_t)br - rw0 * 32u);
    // payload rows of the tile: [t*32 - c0, (t+ntok-1)*32 - cl + flagged(last))
    const uint64_t p0 = (uint64_t)t * 32u - c0;
    const uint64_t p1 = (uint64_t)(t + ntok - 1) * 32u - cl + (uint64_t)__popc(fl_last);
    const uint64_t pa0 = p0 & ~1ull, pa1 = (p1 + 1) & ~1ull;  // 16-byte aligned range
    const bool stage_pay = p1 > p0 && pa1 - pa0 <= (uint64_t)kFlPayRows + 2;
    pay_base[stage] = pa0;
    pay_n[stage] = stage_pay ? (uint32_t)(pa1 - pa0) : 0u;
    const uint32_t pb = stage_pay ? (uint32_t)(pa1 - pa0) * 8u : 0u;
    const uint32_t ib = (uint32_t)(iw1 - iw0) * 4, rb = (uint32_t)(rw1 - rw0) * 4;
    const uint32_t fb = ntok * 4, sb = ntok * 2;
    fence_proxy_async();
    mbar_arrive_expect_tx(&full[stage], ib + rb + 2 * fb + sb + pb);
    if (ib) bulk_g2s(s + g.idx_off, p.idxw + iw0, ib, &full[stage]);
    if (rb) bulk_g2s(s + g.rad_off, p.radw + rw0, rb, &full[stage]);
    bulk_g2s(s + g.fl_off, p.flagw + t, fb, &full[stage]);
    bulk_g2s(s + g.to_off, p.tokoff + t, fb, &full[stage]);
    bulk_g2s(s + g.sc_off, p.scales + t, sb, &full[stage]);
    if (pb) bulk_g2s(s + g.pay_off, p.payloads + pa0 * 4, pb, &full[stage]);
  };

  if (tid == 0) {
    for (int st = 0; st < kFlStages; ++st) {
      mbar_init(&full[st], 1);
      released[st] = 0u;
    }
    mbar_init(&tab_bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  const float4* __restrict__ gtab = reinterpret_cast<const float4*>(p.table) + (int64_t)h * ncw;
  if (tid == 0 && tab_tma) {
    const uint32_t tb = (uint32_t)ncw * 8u;
    fence_proxy_async();
    mbar_arrive_expect_tx(&tab_bar, tb);
    bulk_g2s(tab, p.table16 + (int64_t)h * ncw, tb, &tab_bar);
  }
  pdl_wait();  // the sections come from the encode (PDL)
  pdl_trigger();
  if (tid == 0) {
    int st = 0;
    for (int64_t tile = blockIdx.x; tile < ntile && st < kFlStages; tile += gridDim.x, ++st)
      issue(tile, st);
  }
  if constexpr (!k16) {
    for (int i = tid; i < ncw; i += 256) tab[i] = __ldg(gtab + i);
    __syncthreads();
  } else if (!tab_tma) {
    uint2* t16 = reinterpret_cast<uint2*>(tab);
    for (int i = tid; i < ncw; i += 256) {
      const float4 c = __ldg(gtab + i);
      const __half2 a = __floats2half2_rn(c.x, c.y), b = __floats2half2_rn(c.z, c.w);
      t16[i] = make_uint2(*reinterpret_cast<const uint32_t*>(&a), *reinterpret_cast<const uint32_t*>(&b));
    }
    __syncthreads();
  } else {
    mbar_wait(&tab_bar, 0u);
  }
  const uint32_t imask = w == 32 ? 0xffffffffu : ((1u << w) - 1u);
  const uint32_t rmask = (1u << br) - 1u;
  const float rtop = 1.0f / (float)((1 << br) - 1);
  // lane = (token q of a 4-token group, chunk quad 4*ql .. 4*ql+3): per-token
  // work (flag word, coded offset, scale, run position) is shared by 4 chunks,
  // and the quad's codes are one run read as a 64-bit window
  const int tq = lane >> 3, ql = lane & 7;
  const uint32_t below = (1u << (4 * ql)) - 1u;  // chunks before the quad
  OutT* __restrict__ out = reinterpret_cast<OutT*>(p.out);
  bool bad = false;
  int k = 0;
  for (int64_t tile = blockIdx.x; tile < ntile; tile += gridDim.x, ++k) {
    const int stage = k % kFlStages;
    mbar_wait(&full[stage], (uint32_t)((k / kFlStages) & 1));
    const unsigned char* s = ring + (size_t)stage * g.stage_bytes;
    const uint32_t* iw = reinterpret_cast<const uint32_t*>(s + g.idx_off);
    const uint32_t* rw = reinterpret_cast<const uint32_t*>(s + g.rad_off);
    const uint32_t* fls = reinterpret_cast<const uint32_t*>(s + g.fl_off);
    const uint32_t* tos = reinterpret_cast<const uint32_t*>(s + g.to_off);
    const uint16_t* scs = reinterpret_cast<const uint16_t*>(s + g.sc_off);
    const uint2* pays = reinterpret_cast<const uint2*>(s + g.pay_off);
    // 32-bit arithmetic relative to the tile: coded positions (token offsets
    // are u32), bit offsets from the tile's first code, payload rows mod 2^32
    const uint32_t c0 = tos[0];
    const uint32_t d0i = base_w[stage][0], d0r = base_w[stage][1];  // c0's bit in the staged words
    const uint64_t pbase = pay_base[stage];
    const uint32_t pbase32 = (uint32_t)pbase;
    const uint32_t pn = pay_n[stage];
    const int ntok = (int)min((int64_t)kFlTok, p.nt - tile * kFlTok);
    const uint32_t tok32 = (uint32_t)(tok_base + tile * kFlTok);  // mod 2^32
    OutT* __restrict__ otile = out + (row * p.nt + tile * kFlTok) * 128 + 16 * ql;
#pragma unroll 2
    for (int t4 = 4 * warp; t4 < kFlTok; t4 += 32) {
      const int tt = t4 + tq;
      if (tt < ntok) {
        const uint32_t fw = fls[tt];
        const uint32_t f4 = (fw >> (4 * ql)) & 15u;
        const uint32_t tofs = tos[tt];
        const uint32_t rel0 = tofs - c0 + __popc(~fw & below);  // first coded position of the quad - c0
        const float sg = __half2float(__ushort_as_half(scs[tt])) * rtop;
        const uint32_t ib = rel0 * (uint32_t)w + d0i;
        const uint32_t* ip = iw + (ib >> 5);
        const uint32_t ilo = __funnelshift_r(ip[0], ip[1], ib & 31);
        const uint32_t ihi = __funnelshift_r(ip[1], ip[2], ib & 31);
        const uint64_t iwin = ((uint64_t)ihi << 32) | ilo;  // >= 4 codes of <= 16 bits
        const uint32_t qb = rel0 * (uint32_t)br + d0r;
        const uint32_t qwin = __funnelshift_r(rw[qb >> 5], rw[(qb >> 5) + 1], qb & 31);  // 4 codes <= 8 bits
        float rad[4];
        uint32_t idx[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const uint32_t j = (uint32_t)c - __popc(f4 & ((1u << c) - 1u));  // code slot after skips
          uint32_t ix = (uint32_t)(iwin >> (j * (uint32_t)w)) & imask;
          bad |= !((f4 >> c) & 1u) && ix >= (uint32_t)ncw;  // (a flagged chunk's slot is unused)
          idx[c] = ix < (uint32_t)ncw ? ix : 0u;
          rad[c] = (float)((qwin >> (j * (uint32_t)br)) & rmask) * sg;
        }
        OutT* o = otile + tt * 128;
        if constexpr (std::is_same<OutT, __half>::value) {
          uint2 ov[4];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            ov[c] = mul_round_f16(rad[c], reinterpret_cast<const uint2*>(tab)[idx[c]]);
          }
          // payload row of chunk c = rows before the quad + flagged chunks
          // before c within it (c - slot of c)
          const uint32_t prow0 = (tok32 + (uint32_t)tt) * 32u - tofs + __popc(fw & below) - pbase32;
          if (pn != 0) {  // staged tile: predicated shared loads, no branches
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const uint32_t j = (uint32_t)c - __popc(f4 & ((1u << c) - 1u));
              const uint32_t rel = min(prow0 + (uint32_t)c - j, pn - 1u);
              if ((f4 >> c) & 1u) ov[c] = pays[rel];
            }
          } else if (f4) {  // unstaged tile: the outlier rows from global
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              if ((f4 >> c) & 1u) {
                const uint32_t j = (uint32_t)c - __popc(f4 & ((1u << c) - 1u));
                ov[c] = __ldg(reinterpret_cast<const uint2*>(p.payloads) +
                              (pbase + (uint32_t)(prow0 + (uint32_t)c - j)));
              }
            }
          }
          reinterpret_cast<uint4*>(o)[0] = make_uint4(ov[0].x, ov[0].y, ov[1].x, ov[1].y);
          reinterpret_cast<uint4*>(o)[1] = make_uint4(ov[2].x, ov[2].y, ov[3].x, ov[3].y);
        } else {
          float v[16];
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float4 cw;
            if constexpr (k16) {
              const uint2 h = reinterpret_cast<const uint2*>(tab)[idx[c]];
              const float2 c01 = __half22float2(*reinterpret_cast<const __half2*>(&h.x));
              const float2 c23 = __half22float2(*reinterpret_cast<const __half2*>(&h.y));
              cw = make_float4(c01.x, c01.y, c23.x, c23.y);
            } else {
              cw = tab[idx[c]];
            }
            v[4 * c] = rad[c] * cw.x; v[4 * c + 1] = rad[c] * cw.y;
            v[4 * c + 2] = rad[c] * cw.z; v[4 * c + 3] = rad[c] * cw.w;
          }
          if (f4) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              if ((f4 >> c) & 1u) {
                const uint32_t rel = (tok32 + (uint32_t)tt) * 32u - tofs +
                                     __popc(fw & ((1u << (4 * ql + c)) - 1u)) - pbase32;
                const uint2 hv = rel < pn ? pays[rel]
                                          : __ldg(reinterpret_cast<const uint2*>(p.payloads) + (pbase + rel));
                const float2 a01 = __half22float2(*reinterpret_cast<const __half2*>(&hv.x));
                const float2 a23 = __half22float2(*reinterpret_cast<const __half2*>(&hv.y));
                v[4 * c] = a01.x; v[4 * c + 1] = a01.y; v[4 * c + 2] = a23.x; v[4 * c + 3] = a23.y;
              }
            }
          }
          if constexpr (sizeof(OutT) == 4) {
#pragma unroll
            for (int c = 0; c < 4; ++c)
              reinterpret_cast<float4*>(o)[c] = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
          } else {
            OutT t16[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) t16[i] = Out<OutT>::cvt(v[i]);
            reinterpret_cast<uint4*>(o)[0] = reinterpret_cast<const uint4*>(t16)[0];
            reinterpret_cast<uint4*>(o)[1] = reinterpret_cast<const uint4*>(t16)[1];
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      if (stage_release(&released[stage]) == 7u) {
        released[stage] = 0u;
        const int64_t nxt = tile + (int64_t)kFlStages * gridDim.x;
        if (nxt < ntile) issue(nxt, stage);
      }
    }
  }
  if (bad) atomicOr(p.err, HQMQ_DEVERR_INDEX_RANGE);
}

// Bit-exact fp64 decode: ((q * sigma_w) / top) * codeword (codec.py:315-320).
__global__ void __launch_bounds__(kDecThreads) decode_f64_kernel(DecParams p) {
  const int64_t row = blockIdx.y;
  const int h = (int)((uint32_t)row % (uint32_t)p.H);  // (32-bit: no division subroutine)
  const int ncw = kGroupOrder * p.S;
  const double* __restrict__ tab = reinterpret_cast<const double*>(p.table) + (int64_t)h * ncw * 4;
  const double top = (double)((1 << p.br) - 1);
  const int C = p.C;
  const int64_t nck = p.nt * C;
  double* __restrict__ out = reinterpret_cast<double*>(p.out);
  for (int64_t ci = (int64_t)blockIdx.x * kDecThreads + threadIdx.x; ci < nck;
       ci += (int64_t)gridDim.x * kDecThreads) {
    const int64_t tr = ci / C;
    const int c = (int)(ci - tr * C);
    const int64_t tok = row * p.T + p.t0 + tr;
    bool fl;
    const uint64_t pos = coded_pos(p, tok, c, fl);
    double v[4];
    if (!fl) {
      uint32_t idx = read_bits(p.idxw, pos * (uint64_t)p.w, p.w);
      const uint32_t q = read_bits(p.radw, pos * (uint64_t)p.br, p.br);
      if (idx >= (uint32_t)ncw) {
        atomicOr(p.err, HQMQ_DEVERR_INDEX_RANGE);
        idx = 0;
      }
      const double sw = (double)__half2float(__ushort_as_half(__ldg(p.scales + tok)));
      const double rad = __ddiv_rn(__dmul_rn((double)q, sw), top);
#pragma unroll
      for (int i = 0; i < 4; ++i) v[i] = __dmul_rn(rad, __ldg(tab + 4 * (int64_t)idx + i));
    } else {
      const uint64_t prow = (uint64_t)tok * C + c - pos;
      const ushort4 hv = __ldg(reinterpret_cast<const ushort4*>(p.payloads) + prow);
      v[0] = (double)__half2float(__ushort_as_half(hv.x));
      v[1] = (double)__half2float(__ushort_as_half(hv.y));
      v[2] = (double)__half2float(__ushort_as_half(hv.z));
      v[3] = (double)__half2float(__ushort_as_half(hv.w));
    }
    double* o = out + (row * p.nt + tr) * p.D + 4 * c;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (4 * c + i < p.D) o[i] = v[i];
  }
}

__global__ void unpack_kernel(DecParams p, int32_t* indices, uint8_t* quanta, uint8_t* flags) {
  const int64_t n = p.B * p.H * p.T * p.C;
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x) {
    const int64_t tok = g / p.C;
    const int c = (int)(g - tok * p.C);
    bool fl;
    const uint64_t pos = coded_pos(p, tok, c, fl);
    if (fl) {
      indices[g] = 0;
      quanta[g] = 0;
    } else {
      indices[g] = (int32_t)read_bits(p.idxw, pos * (uint64_t)p.w, p.w);
      quanta[g] = (uint8_t)read_bits(p.radw, pos * (uint64_t)p.br, p.br);
    }
    flags[g] = fl ? 1 : 0;
  }
}

__global__ void coded_mark_kernel(int64_t n, const uint8_t* flags, uint32_t* mark) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x)
    mark[g] = flags && flags[g] ? 0u : 1u;
}

__global__ void pack_kernel(int64_t n, int C, int w, int br, const int32_t* indices,
                            const uint8_t* quanta, const uint8_t* flags, const uint32_t* pos,
                            uint32_t* idxw, uint32_t* radw, uint32_t* flagw, uint32_t* tokoff) {
  for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < n;
       g += (int64_t)gridDim.x * blockDim.x) {
    const bool fl = flags && flags[g];
    const uint64_t ps = pos[g];
    if (tokoff && (g % C) == 0) tokoff[g / C] = (uint32_t)ps;
    if (fl) {
      atomicOr(flagw + (g >> 5), 1u << (g & 31));
      continue;
    }
    const uint32_t iv = (uint32_t)indices[g];
    const uint64_t bi = ps * (uint64_t)w;
    atomicOr(idxw + (bi >> 5), iv << (bi & 31));
    if ((bi & 31) + w > 32) atomicOr(idxw + (bi >> 5) + 1, iv >> (32 - (bi & 31)));
    const uint32_t qv = (uint32_t)quanta[g];
    const uint64_t br_ = ps * (uint64_t)br;
    atomicOr(radw + (br_ >> 5), qv << (br_ & 31));
    if ((br_ & 31) + br > 32) atomicOr(radw + (br_ >> 5) + 1, qv >> (32 - (br_ & 31)));
  }
}

__global__ void token_coded_kernel(int64_t n_tokens, int C, const uint32_t* flagw, uint32_t* cnt) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_tokens;
       t += (int64_t)gridDim.x * blockDim.x) {
    uint64_t b = (uint64_t)t * C;
    const uint64_t e = b + C;
    uint32_t nflag = 0;
    while (b < e) {
      const uint32_t word = __ldg(flagw + (b >> 5));
      const uint32_t sh = (uint32_t)(b & 31);
      const uint64_t take = min((uint64_t)(32 - sh), e - b);
      const uint32_t m = take == 32 ? 0xffffffffu : ((1u << take) - 1u);
      nflag += __popc((word >> sh) & m);
      b += take;
    }
    cnt[t] = (uint32_t)C - nflag;
  }
}

__global__ void validate_kernel(const uint32_t* idxw, int64_t n, int w, int64_t limit,
                                uint32_t* err) {
  bool bad = false;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= (int64_t)read_bits(idxw, (uint64_t)i * w, w) >= limit;
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, HQMQ_DEVERR_INDEX_RANGE);
}

namespace {
int check() { return check_launch(); }
int grid_for(int64_t n, int threads) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, threads), 148 * 16));
}

bool fill(const hqmq_decode_args* a, DecParams& p, bool need_range) {
  if (!a || a->batch < 1 || a->heads < 1 || a->tokens < 0 || a->head_dim < 1) return false;
  if (a->codebook_size < 1 || a->radius_bits < 1 || a->radius_bits > 8 || a->index_bits < 1 ||
      a->index_bits > 32)
    return false;
  if (need_range && !(0 <= a->token_start && a->token_start <= a->token_stop &&
                      a->token_stop <= a->tokens))
    return false;
  p.B = a->batch; p.H = a->heads; p.T = a->tokens; p.D = a->head_dim;
  p.C = (int)ceil_div(a->head_dim, 4);
  p.S = a->codebook_size; p.br = a->radius_bits; p.w = a->index_bits;
  p.t0 = a->token_start; p.nt = a->token_stop - a->token_start;
  p.scales = a->scales; p.idxw = a->index_words; p.radw = a->radius_words;
  p.flagw = a->flag_words; p.payloads = a->payloads; p.tokoff = a->token_offsets;
  p.out = a->out; p.err = a->error_word;
  p.table16 = reinterpret_cast<const uint2*>(a->joint_f16);
  return true;
}

// CTAs per row for a persistent-style launch over ntile tiles per row: as many
// as are co-resident in ONE wave (occupancy query, cached per kernel / smem /
// device), so that no CTA waits for a second wave while the rest idle.
template <typename K>
int64_t one_wave_ctas_per_row(K kern, size_t smem, int64_t rows, int64_t ntile) {
  struct Entry {
    const void* k;
    size_t smem;
    int dev, slots;
  };
  static thread_local Entry cache[8] = {};
  static thread_local int next = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  // the whole unified L1 / shared array as shared memory, so that the
  // occupancy the grid is sized for is the one the launch gets
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                       (int)cudaSharedmemCarveoutMaxShared);
  int slots = 0;
  for (const Entry& e : cache)
    if (e.k == reinterpret_cast<const void*>(kern) && e.smem == smem && e.dev == dev) slots = e.slots;
  if (!slots) {
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    slots = std::max(1, per_sm) * std::max(1, sms);
    cache[next] = Entry{reinterpret_cast<const void*>(kern), smem, dev, slots};
    next = (next + 1) % 8;
  }
  return std::max<int64_t>(1, std::min<int64_t>(slots / rows, ntile));
}

template <typename OutT>
int launch_decode(DecParams& p, const hqmq_decode_args* a, cudaStream_t st) {
  const int64_t rows = p.B * p.H;
  const size_t smem = (size_t)kGroupOrder * p.S * sizeof(float4);
  const bool use_smem = smem <= kDecSmemLimit;
  p.table = a->joint_f32;
  p.aligned4 = (p.D % 4 == 0) && (reinterpret_cast<uintptr_t>(a->out) % (4 * sizeof(OutT)) == 0);
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (p.D == 128 && p.flagw && p.tokoff && p.payloads && use_smem && p.aligned4 && p.w <= 16 &&
      p.T % 8 == 0 && p.t0 % 8 == 0 && p.nt % 8 == 0 && al16(p.idxw) && al16(p.radw) &&
      al16(p.scales) && al16(p.flagw) && al16(p.tokoff)) {
    const FlagGeom g = fl_geom(p.w, p.br);
    const size_t fsmem = fd_table_bytes<OutT>(kGroupOrder * p.S) + (size_t)kFlStages * g.stage_bytes;
    cudaFuncSetAttribute(decode_flag_tma_kernel<OutT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    void (*kern)(DecParams) = decode_flag_tma_kernel<OutT>;
    switch (p.w * 16 + p.br) {
      case 9 * 16 + 4: kern = decode_flag_tma_kernel<OutT, 9, 4>; break;    // C1: S = 16
      case 11 * 16 + 4: kern = decode_flag_tma_kernel<OutT, 11, 4>; break;  // S = 64
      case 11 * 16 + 6: kern = decode_flag_tma_kernel<OutT, 11, 6>; break;  // C3: S = 64, b_r 6
      case 13 * 16 + 4: kern = decode_flag_tma_kernel<OutT, 13, 4>; break;  // S = 256
      default: break;
    }
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int64_t bx = one_wave_ctas_per_row(kern, fsmem, rows, ceil_div(p.nt, kFlTok));
    const cudaError_t e = launch_pdl(kern, dim3((unsigned)bx, (unsigned)rows), dim3(256), fsmem, st, p);
    return e == cudaSuccess ? check() : record_cuda_error(e);
  }
  if (p.D == 128 && p.flagw && p.tokoff && p.payloads && use_smem && p.aligned4) {
    const int64_t nwt = ceil_div(p.nt, 32);  // 8 warps x 4 tokens per CTA step
    const int64_t want = std::max<int64_t>(1, ceil_div((int64_t)148 * 4, rows));
    const int64_t bx = std::max<int64_t>(1, std::min<int64_t>(want, nwt));
    cudaFuncSetAttribute(decode_flag_kernel<OutT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kDecSmemLimit);
    decode_flag_kernel<OutT><<<dim3((unsigned)bx, (unsigned)rows), 256,
                               fd_table_bytes<OutT>(kGroupOrder * p.S), st>>>(p);
    return check();
  }
  const bool fast = p.D == 128 && !p.flagw && use_smem && p.aligned4 && p.T % 8 == 0 &&
                    p.t0 % 8 == 0 && p.nt % 8 == 0 && al16(p.idxw) && al16(p.radw) &&
                    al16(p.scales);
  if (fast) {
    const FastDecodeGeom g = fd_geom(p.w, p.br);
    const size_t fsmem = fd_table_bytes<OutT>(kGroupOrder * p.S) + (size_t)kFDStages * g.stage_bytes;
    // (index_bits, radius_bits) instances with compile-time stream geometry
    void (*kern)(DecParams) = decode_fast_kernel<OutT, 0, 0>;
    switch (p.w * 16 + p.br) {
      case 9 * 16 + 4: kern = decode_fast_kernel<OutT, 9, 4>; break;    // S = 16
      case 11 * 16 + 4: kern = decode_fast_kernel<OutT, 11, 4>; break;  // S = 64
      case 13 * 16 + 4: kern = decode_fast_kernel<OutT, 13, 4>; break;  // S = 256
      case 11 * 16 + 6: kern = decode_fast_kernel<OutT, 11, 6>; break;  // Qwen b_r 6
      default: break;
    }
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int64_t bx = one_wave_ctas_per_row(kern, fsmem, rows, ceil_div(p.nt, kFDTok));
    const cudaError_t e = launch_pdl(kern, dim3((unsigned)bx, (unsigned)rows), dim3(256), fsmem, st, p);
    return e == cudaSuccess ? check() : record_cuda_error(e);
  }
  const int64_t nck = p.nt * p.C;
  const int64_t want = std::max<int64_t>(1, (148 * 4 + rows - 1) / rows);
  const int64_t bx = std::max<int64_t>(1, std::min<int64_t>(want, ceil_div(nck, kDecThreads * kDecR)));
  const dim3 grid((unsigned)bx, (unsigned)rows);
  if (use_smem) {
    // set on every launch: the attribute is per device, and a process may drive several
    cudaFuncSetAttribute(decode_kernel<OutT, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kDecSmemLimit);
    decode_kernel<OutT, true><<<grid, kDecThreads, smem, st>>>(p);
  } else {
    decode_kernel<OutT, false><<<grid, kDecThreads, 0, st>>>(p);
  }
  return check();
}

// Med3x compact layout -> fixed per-token code slots (the paged cache's
// layout): warp = token, lane = chunk (head_dim 128).  Token t's index codes
// go to bits [32*w*t + lane*w, +w) of `islots` (w words per token), radius
// codes likewise; a flagged chunk's slot is 0.  payoff[t] = payload_base +
// the token's first payload row (t*32 - token_offsets[t]).
__global__ void __launch_bounds__(256) expand_kernel(DecParams p, uint32_t* __restrict__ islots,
                                                     uint32_t* __restrict__ rslots,
                                                     uint32_t* __restrict__ payoff,
                                                     uint32_t payload_base, int64_t ntok) {
  __shared__ uint32_t sw[8][16 + 8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int w = p.w, br = p.br;
  for (int64_t tok = (int64_t)blockIdx.x * 8 + warp; tok < ntok; tok += (int64_t)gridDim.x * 8) {
    const uint32_t fw = __ldg(p.flagw + tok);
    const bool fl = (fw >> lane) & 1u;
    const uint32_t base = __ldg(p.tokoff + tok);
    const uint64_t pos = (uint64_t)base + lane - __popc(fw & ((1u << lane) - 1u));
    const uint32_t idx = fl ? 0u : read_bits(p.idxw, pos * (uint64_t)w, w);
    const uint32_t q = fl ? 0u : read_bits(p.radw, pos * (uint64_t)br, br);
    if (lane < 24) sw[warp][lane] = 0u;
    __syncwarp();
    auto put = [&](uint32_t* dst, uint32_t v, int width) {
      const uint32_t bit = (uint32_t)lane * width;
      atomicOr(dst + (bit >> 5), v << (bit & 31));
      if ((bit & 31) + width > 32) atomicOr(dst + (bit >> 5) + 1, v >> (32 - (bit & 31)));
    };
    put(sw[warp], idx, w);
    put(sw[warp] + 16, q, br);
    __syncwarp();
    if (lane < w) islots[tok * w + lane] = sw[warp][lane];
    if (lane < br) rslots[tok * br + lane] = sw[warp][16 + lane];
    if (lane == 0) payoff[tok] = payload_base + (uint32_t)(tok * 32 - (int64_t)base);
    __syncwarp();
  }
}
}  // namespace

// Prefill: decode a whole no-Med3x tensor to fp16 straight into UMMA tiles of
// 2^tile_log2 keys (K-major or MN-major), ntk tiles per (batch, head) row.
// Returns HQMQ_ERR_UNSUPPORTED when the fast decode does not apply (the
// caller then decodes row-major and re-lays the result out).
int decode_fp16_tiles(const hqmq_decode_args* a, int tile_log2, int mn, int64_t ntk, void* tiles,
                      cudaStream_t st) {
  DecParams p;
  if (!fill(a, p, true) || a->out_dtype != HQMQ_F16 || p.t0 != 0 || p.nt != p.T)
    return HQMQ_ERR_UNSUPPORTED;
  if (p.B * p.H >= 65536 || p.nt == 0) return HQMQ_ERR_UNSUPPORTED;
  auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  const size_t smem = (size_t)kGroupOrder * p.S * sizeof(float4);
  const bool fast = p.D == 128 && !p.flagw && smem <= kDecSmemLimit && p.T % 8 == 0 &&
                    al16(p.idxw) && al16(p.radw) && al16(p.scales) && al16(tiles);
  if (!fast) return HQMQ_ERR_UNSUPPORTED;
  p.aligned4 = 1;
  p.out = tiles;
  p.tile_log2 = tile_log2;
  p.tile_mn = mn;
  p.tile_ntk = ntk;
  const int64_t rows = p.B * p.H;
  const FastDecodeGeom g = fd_geom(p.w, p.br);
  const size_t fsmem = fd_table_bytes<__half>(kGroupOrder * p.S) + (size_t)kFDStages * g.stage_bytes;
  void (*kern)(DecParams) = decode_fast_kernel<__half, 0, 0, true>;
  switch (p.w * 16 + p.br) {
    case 9 * 16 + 4: kern = decode_fast_kernel<__half, 9, 4, true>; break;
    case 11 * 16 + 4: kern = decode_fast_kernel<__half, 11, 4, true>; break;
    case 13 * 16 + 4: kern = decode_fast_kernel<__half, 13, 4, true>; break;
    case 11 * 16 + 6: kern = decode_fast_kernel<__half, 11, 6, true>; break;
    default: break;
  }
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  const int64_t bx = one_wave_ctas_per_row(kern, fsmem, rows, ceil_div(p.nt, kFDTok));
  kern<<<dim3((unsigned)bx, (unsigned)rows), 256, fsmem, st>>>(p);
  return check();
}
}  // namespace hqmq

namespace hqmq {
// Paged append scatter (hqmq_paged_append): warp = one source token row.
__global__ void __launch_bounds__(256) paged_append_kernel(hqmq_paged_append_args a, int64_t n_rows) {
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * 8;
  for (int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); r < n_rows; r += stride) {
    const int64_t t = r % a.n_new, ih = r / a.n_new;
    const int h = (int)(ih % a.kv_heads), i = (int)(ih / a.kv_heads);
    const int64_t pos = (int64_t)__ldg(a.seq_start + i) + t;
    const int64_t pi = pos / a.page_tokens, o = pos - pi * a.page_tokens;
    const int64_t page = pi < a.max_pages
        ? (int64_t)__ldg(a.block_table + ((int64_t)__ldg(a.seq_ids + i) * a.kv_heads + h) * a.max_pages + pi)
        : -1;
    if (page < 0 || page >= a.num_pages) {
      if (lane == 0 && a.error_word) atomicOr(a.error_word, HQMQ_DEVERR_INDEX_RANGE);
      continue;
    }
    const int64_t slot = page * a.page_tokens + o;
    if (lane < a.index_bits)
      a.index_pages[slot * a.index_bits + lane] = __ldg(a.src_index + r * a.index_bits + lane);
    if (lane < a.radius_bits)
      a.radius_pages[slot * a.radius_bits + lane] = __ldg(a.src_radius + r * a.radius_bits + lane);
    if (lane == 0) a.scale_pages[slot] = __ldg(a.src_scales + r);
    if (a.flag_pages) {
      if (lane == 1) a.flag_pages[slot] = __ldg(a.src_flags + r);
      if (lane == 2) a.payoff_pages[slot] = __ldg(a.src_payoff + r);
    }
  }
}
}  // namespace hqmq

extern "C" {

int hqmq_decode(const hqmq_decode_args* a, void* stream) {
  using namespace hqmq;
  DecParams p;
  if (!fill(a, p, true)) return HQMQ_ERR_INVALID_ARGUMENT;
  if (p.B * p.H >= 65536) return HQMQ_ERR_UNSUPPORTED;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (p.nt == 0) return HQMQ_OK;
  switch (a->out_dtype) {
    case HQMQ_F32: return launch_decode<float>(p, a, st);
    case HQMQ_F16: return launch_decode<__half>(p, a, st);
    case HQMQ_BF16: return launch_decode<__nv_bfloat16>(p, a, st);
    case HQMQ_F64: {
      p.table = a->joint_f64;
      const int64_t rows = p.B * p.H;
      const int64_t bx = std::max<int64_t>(1, std::min<int64_t>(64, ceil_div(p.nt * p.C, kDecThreads)));
      decode_f64_kernel<<<dim3((unsigned)bx, (unsigned)rows), kDecThreads, 0, st>>>(p);
      return check();
    }
    default: return HQMQ_ERR_INVALID_ARGUMENT;
  }
}

int hqmq_paged_append(const hqmq_paged_append_args* a, void* stream) {
  using namespace hqmq;
  if (!a || a->n_seq < 0 || a->kv_heads < 1 || a->n_new < 0 || a->max_pages < 1 ||
      a->page_tokens < 1 || a->index_bits < 1 || a->index_bits > 32 || a->radius_bits < 1 ||
      a->radius_bits > 32 || a->num_pages < 1 || !a->seq_ids || !a->seq_start || !a->block_table ||
      !a->src_index || !a->src_radius || !a->src_scales || !a->index_pages || !a->radius_pages ||
      !a->scale_pages)
    return HQMQ_ERR_INVALID_ARGUMENT;
  if ((a->flag_pages != nullptr) != (a->payoff_pages != nullptr) ||
      (a->flag_pages && (!a->src_flags || !a->src_payoff)))
    return HQMQ_ERR_INVALID_ARGUMENT;
  const int64_t n_rows = (int64_t)a->n_seq * a->kv_heads * a->n_new;
  if (n_rows == 0) return HQMQ_OK;
  const int64_t blocks = std::min<int64_t>(ceil_div(n_rows, 8), 148 * 8);
  paged_append_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(*a, n_rows);
  return check();
}

int hqmq_expand_tokens(const hqmq_decode_args* a, uint32_t* index_slots, uint32_t* radius_slots,
                       uint32_t* payload_offsets, uint32_t payload_base, void* stream) {
  using namespace hqmq;
  DecParams p;
  if (!fill(a, p, false)) return HQMQ_ERR_INVALID_ARGUMENT;
  if (p.D != 128 || !p.flagw || !p.tokoff || p.w > 16 || p.br > 8 || !index_slots ||
      !radius_slots || !payload_offsets)
    return HQMQ_ERR_INVALID_ARGUMENT;
  const int64_t ntok = p.B * p.H * p.T;
  if (ntok == 0) return HQMQ_OK;
  const int64_t blocks = std::min<int64_t>(ceil_div(ntok, 8), 148 * 16);
  expand_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      p, index_slots, radius_slots, payload_offsets, payload_base, ntok);
  return check();
}

int hqmq_unpack(const hqmq_decode_args* a, int32_t* indices, uint8_t* quanta, uint8_t* flags,
                void* stream) {
  using namespace hqmq;
  DecParams p;
  if (!fill(a, p, false)) return HQMQ_ERR_INVALID_ARGUMENT;
  const int64_t n = p.B * p.H * p.T * p.C;
  if (n == 0) return HQMQ_OK;
  unpack_kernel<<<grid_for(n, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      p, indices, quanta, flags);
  return check();
}

size_t hqmq_pack_workspace_bytes(int64_t n_chunks) {
  if (n_chunks >= (1LL << 31)) return 0;
  size_t cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                (int)std::max<int64_t>(n_chunks, 1));
  return ((size_t)std::max<int64_t>(n_chunks, 1) * 4 * 2 + 255) / 256 * 256 + cub_bytes;
}

int hqmq_pack(int64_t n, int32_t C, int32_t w, int32_t br, const int32_t* indices,
              const uint8_t* quanta, const uint8_t* flags, uint32_t* idxw, uint32_t* radw,
              uint32_t* flagw, uint32_t* tokoff, void* workspace, size_t workspace_bytes,
              void* stream) {
  using namespace hqmq;
  if (n < 0 || C < 1 || w < 1 || w > 32 || br < 1 || br > 8) return HQMQ_ERR_INVALID_ARGUMENT;
  // cub's scan takes an int item count: keep n below 2^31 (a single
  // (layer, role) call that large would be 17 GB of fp16 input)
  if (n >= (1LL << 31)) return HQMQ_ERR_UNSUPPORTED;
  if (workspace_bytes < hqmq_pack_workspace_bytes(n)) return HQMQ_ERR_WORKSPACE;
  if (n == 0) return HQMQ_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  char* ws = reinterpret_cast<char*>(workspace);
  uint32_t* mark = reinterpret_cast<uint32_t*>(ws);
  uint32_t* pos = mark + n;
  char* tmp = ws + ((size_t)n * 8 + 255) / 256 * 256;
  size_t tmp_bytes = workspace_bytes - (size_t)(tmp - ws);
  coded_mark_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, flags, mark);
  {
    const cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, mark, pos, (int)n, st);
    if (e != cudaSuccess) return record_cuda_error(e);
  }
  pack_kernel<<<grid_for(n, 256), 256, 0, st>>>(n, C, w, br, indices, quanta, flags, pos, idxw,
                                                  radw, flags ? flagw : nullptr,
                                                  flags ? tokoff : nullptr);
  return check();
}

size_t hqmq_token_offsets_workspace_bytes(int64_t n_tokens) {
  if (n_tokens >= (1LL << 31)) return 0;
  size_t cub_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, (const uint32_t*)nullptr, (uint32_t*)nullptr,
                                (int)std::max<int64_t>(n_tokens, 1));
  return ((size_t)std::max<int64_t>(n_tokens, 1) * 4 + 255) / 256 * 256 + cub_bytes;
}

int hqmq_token_offsets(int64_t n_tokens, int32_t C, const uint32_t* flagw, uint32_t* tokoff,
                       void* workspace, size_t workspace_bytes, void* stream) {
  using namespace hqmq;
  if (n_tokens < 0 || C < 1) return HQMQ_ERR_INVALID_ARGUMENT;
  if (n_tokens >= (1LL << 31)) return HQMQ_ERR_UNSUPPORTED;  // cub int item count
  if (workspace_bytes < hqmq_token_offsets_workspace_bytes(n_tokens)) return HQMQ_ERR_WORKSPACE;
  if (n_tokens == 0) return HQMQ_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  char* ws = reinterpret_cast<char*>(workspace);
  uint32_t* cnt = reinterpret_cast<uint32_t*>(ws);
  char* tmp = ws + ((size_t)n_tokens * 4 + 255) / 256 * 256;
  size_t tmp_bytes = workspace_bytes - (size_t)(tmp - ws);
  token_coded_kernel<<<grid_for(n_tokens, 256), 256, 0, st>>>(n_tokens, C, flagw, cnt);
  const cudaError_t e = cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, cnt, tokoff, (int)n_tokens, st);
  if (e != cudaSuccess) return record_cuda_error(e);
  return check();
}

int hqmq_validate_indices(const uint32_t* idxw, int64_t n, int32_t w, int64_t limit,
                          uint32_t* err, void* stream) {
  using namespace hqmq;
  if (n < 0 || w < 1 || w > 32) return HQMQ_ERR_INVALID_ARGUMENT;
  if (n == 0) return HQMQ_OK;
  validate_kernel<<<grid_for(n, 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      idxw, n, w, limit, err);
  return check();
}

}  // extern "C"
