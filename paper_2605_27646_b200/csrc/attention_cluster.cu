// Decode attention over the compressed cache as a CTA PAIR (a thread-block
// cluster of 2 on two SMs): one CTA owns the K side, the other the V side.
//
// Reference path replaced: attention.fused_attend (attention.py:137-199) for
// decode steps (T_q x GQA group <= 8 query rows per kv head), head_dim 128,
// without outlier extraction, S <= 64 (the C4 configuration).
//
// Why a pair.  Every (key, chunk) of K and V is decoded by a random gather
// from its (layer, kv head, role) joint table (24 S codewords, codec.py:
// 315-320).  A gather from ONE copy of the table costs ~6.2 shared-memory
// wavefronts per warp (bank conflicts; ncu of the single-CTA kernel,
// profiles/r02_ncu_attn_mma.txt) against 2 for a conflict-free 64-bit access.
// Sixteen replicas of the table, replica j confined to bank pair j (entry e
// of replica j at byte 128 e + 8 j) and lane l reading replica l % 16, make
// every half-warp's gathers hit 16 distinct bank pairs: 2 wavefronts.  At
// S = 64 that is 1536 x 128 B = 192 KB -- one role's table per SM.  So the
// K CTA holds the replicated K table and the V CTA the V table.
//
// Work = items (kv head, sequence, key split), hkv-major so a CTA reloads its
// table at most a couple of times; the clusters take contiguous item ranges
// (persistent).  Inside an item each of the 16 warps of a CTA streams its own
// 16-key blocks (block j of the item goes to warp j % 16): the next block's
// code words are loaded into registers (L1/L2, prefetched into L2 a few
// blocks ahead) while the current one is decoded, so no CTA-wide pipeline or
// barrier sits on the hot path.  Warp w of the K CTA and warp w of the V CTA
// walk the same blocks:
//
//   K warp: decodes its block's 16 keys straight into mma.sync A fragments
//           (S^T = K Q^T, m16n8k16: M = 16 keys, N = the <= 8 query rows, K =
//           16 permuted dims = 4 chunks per slab), runs the online softmax
//           (log2 domain, per-key sigma folded in, the running max raised
//           only when a block exceeds it by more than 8 so most blocks need
//           no rescale), and st.async-es the fp16 P and the row rescale
//           factors (288 bytes) into its V twin's mailbox in the V CTA,
//           completion counted on the twin's mbarrier (DSMEM, no fence);
//   V warp: decodes its block's V chunks into mma.sync A fragments and
//           accumulates O^T += V^T P^T (M = 16 dims, N = rows, K = 16 keys),
//           rescaling O only when a factor is not 1, and frees the mailbox
//           with a relaxed remote arrive.
// Per (item, warp) the K CTA writes the partial (m, l) and the V CTA the
// partial O; combine_kernel merges them (and applies the deferred 2^9 / top).
#include <algorithm>
#include <cstdint>
#include <cmath>

#include "attention.cuh"

namespace hqmq {
namespace {

constexpr int kBK = 16;                     // keys per warp block
constexpr int kCW = 16;                     // warps per CTA
constexpr int kCThreads = kCW * 32;
#ifndef HQMQ_PAIR_PF
#define HQMQ_PAIR_PF 0
#endif
constexpr int kPfDist = HQMQ_PAIR_PF;       // L2 prefetch distance (own blocks ahead)
constexpr float kLazy = 8.0f;               // raise the running max only past this margin (log2)
// K -> V message per warp and block: P as fp16 [8 rows][16 keys] (key k at
// position 2 (k % 8) + k / 8) and the 8 rows' rescale factors (fp32)
constexpr uint32_t kMsgP = 8 * 16 * 2;
constexpr uint32_t kWarpMsg = kMsgP + 8 * 4;
constexpr size_t kSmemMax = 232448;
constexpr int kNcMax = 74;                  // clusters (148 SMs / 2) the item split assumes
constexpr int kMaxCw = 1536;                // S <= 64
constexpr size_t kTab = (size_t)kMaxCw * 128;
constexpr size_t kBoxOff = kTab;                         // mailboxes (V CTA)
constexpr size_t kBarOff = kBoxOff + (size_t)kCW * kWarpMsg;
constexpr size_t kSmem = kBarOff + kCW * 8;
static_assert(kSmem <= kSmemMax, "pair attention shared memory");

struct CParams {
  AttParams p;
  int nsplit;               // key splits per row
  int64_t kps;              // keys per split (multiple of 128)
  int64_t items;            // Hkv * B * nsplit, hkv-major (< 2^31)
  int ncw;
  float q_scale;            // softmax scale * log2(e) * 2^9 / top, from the host
  // (the kernel's loop is kept free of subroutine calls -- 64-bit integer and
  // IEEE fp32 division -- so ptxas keeps the global-memory descriptor in
  // uniform registers instead of re-materialising it before every load)
};

// ---------------------------------------------------------------- PTX bits
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" :::
                   "memory");
}
// bytes into the peer CTA's shared memory, completion counted on the peer's mbarrier
__device__ __forceinline__ void st_async4(uint32_t raddr, uint32_t rbar, uint32_t a) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(raddr),
               "r"(a), "r"(rbar)
               : "memory");
}
__device__ __forceinline__ void st_async8(uint32_t raddr, uint32_t rbar, uint32_t a, uint32_t b) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];" ::"r"(
                   raddr),
               "r"(a), "r"(b), "r"(rbar)
               : "memory");
}
// mailbox-free signal to the peer: relaxed (a release would fence the whole
// GPU memory system, MEMBAR.ALL.GPU); callers issue it only after the
// mailbox's loaded values are in registers, which orders the reads first
__device__ __forceinline__ void remote_arrive(uint32_t rbar) {
  asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
__device__ __forceinline__ uint2 lds64(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr));
  return v;
}
// 2^x on the MUFU (flushes denormal results to 0: fine for softmax weights)
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t hmul2_raw(uint32_t a, uint32_t b) {
  uint32_t r;
  asm("mul.rn.f16x2 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
  return r;
}
// non-volatile mma: the compiler may interleave them with the decode
__device__ __forceinline__ void mma_f(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                      uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// ------------------------------------------------------------ decode bits
// The replicated table holds the fp16 codewords scaled by 2^15, and the
// radius code q enters the product as the fp16 DENORMAL q * 2^-24 (its bits
// are q itself: no int->float conversion), so r * c comes out as
// q * c * 2^-9 (exact fp16 product, normal for q * |c| >= 2^-5; below that
// the absolute error stays under 2^-24 * 2^9 = 3e-5 of the unscaled value).
// The 2^9 / top factor is folded into Q (scores) and into the combine (O).
constexpr float kProdScale = 512.0f;  // 2^9

// N index codes of W bits, aligned once by runtime funnel shifts (the run's
// in-word shift depends on the lane); each code's TABLE BYTE OFFSET
// (code * 128, the entry stride of the replicated table) then comes out of
// one funnel shift + one AND (+ the lane's replica base).
template <int N, int W, int NT>
struct IdxRun {
  static constexpr int kSpan = max_run_shift(N, W, NT) + N * W;
  static constexpr int kNW = (kSpan + 31) / 32;
  uint32_t r[kNW];
  __device__ __forceinline__ void align(const uint32_t (&w)[kNW], uint32_t sh) {
#pragma unroll
    for (int i = 0; i < kNW; ++i) r[i] = __funnelshift_r(w[i], i + 1 < kNW ? w[i + 1] : 0u, sh);
  }
  __device__ __forceinline__ uint32_t addr(int i, uint32_t tab_lane) const {
    constexpr uint32_t kMask = ((1u << W) - 1u) << 7;
    const int b = i * W - 7;
    uint32_t x;
    if (b < 0) {
      x = r[0] << (-b);
    } else {
      const int wi = b >> 5, sh = b & 31;
      x = sh == 0 ? r[wi] : __funnelshift_r(r[wi], wi + 1 < kNW ? r[wi + 1] : 0u, sh);
    }
    return (x & kMask) + tab_lane;
  }
};

// (q, q) as fp16 denormals from byte K of `src` (q in its low nibble), b_r = 4
template <int K>
__device__ __forceinline__ uint32_t rad4(uint32_t src) {
  return __byte_perm(src, 0u, (uint32_t)(K | (4 << 4) | (K << 8) | (4 << 12))) & 0x000F000Fu;
}
__device__ __forceinline__ uint32_t radq(uint32_t q) { return q * 0x10001u; }  // q < 2^8

// replicate the joint table (fp16 codewords x 2^15) 16 times: entry e of
// replica j at byte 128 e + 8 j (4 source loads in flight per thread)
__device__ __forceinline__ void fill_table(uint2* tab, const uint2* __restrict__ src, int ncw, int tid) {
  const int lane = tid & 31, w = tid >> 5;
  const uint32_t s15 = 0x78007800u;  // (32768, 32768) fp16
  constexpr int kStep = 2 * kCW;
  for (int e0 = 2 * w + (lane >> 4); e0 < ncw; e0 += 4 * kStep) {
    uint2 v[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) v[k] = e0 + k * kStep < ncw ? __ldg(src + e0 + k * kStep) : make_uint2(0u, 0u);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (e0 + k * kStep < ncw)
        tab[(e0 + k * kStep) * 16 + (lane & 15)] = make_uint2(hmul2_raw(v[k].x, s15), hmul2_raw(v[k].y, s15));
  }
}

// one item = (kv head, sequence, key split), hkv-major
struct Item {
  int64_t bh, b, hkv, kbeg;
  int kend_rel, nblk, split;
};
__device__ __forceinline__ Item item_at(const CParams& c, int64_t i) {
  const AttParams& p = c.p;
  Item it;
  const uint32_t per_h = (uint32_t)p.B * (uint32_t)c.nsplit;  // 32-bit: items < 2^31
  const uint32_t hk = (uint32_t)i / per_h;
  const uint32_t r = (uint32_t)i - hk * per_h;
  const uint32_t bq = r / (uint32_t)c.nsplit;
  it.hkv = hk;
  it.b = bq;
  it.split = (int)(r - bq * (uint32_t)c.nsplit);
  it.bh = it.b * p.Hkv + it.hkv;
  const int64_t tkv = p.kv_lens ? (int64_t)__ldg(p.kv_lens + it.b) : p.Tkv;
  it.kbeg = (int64_t)it.split * c.kps;
  const int64_t kend = min(tkv, it.kbeg + c.kps);
  it.kend_rel = kend > it.kbeg ? (int)(kend - it.kbeg) : 0;
  it.nblk = (int)ceil_div(it.kend_rel, kBK);
  return it;
}

// token index (in the section streams) of item-relative key `k`
template <bool kPaged>
__device__ __forceinline__ int64_t token_of(const AttParams& p, const Item& it, int k) {
  const int64_t key = it.kbeg + k;
  if constexpr (kPaged)
    return (int64_t)__ldg(p.block_table + it.bh * p.max_pages + key / 128) * 128 + (key & 127);
  else
    return it.bh * p.Tkv + key;
}

// the page id of item-relative block jb (paged caches), loaded a block ahead
// of its code words so that the table read is off the code loads' critical path
template <bool kPaged>
__device__ __forceinline__ int32_t block_page(const AttParams& p, const Item& it, int jb) {
  if constexpr (kPaged)
    return __ldg(p.block_table + it.bh * p.max_pages + (it.kbeg + (int64_t)jb * kBK) / 128);
  else
    return 0;
}
template <bool kPaged>
__device__ __forceinline__ int64_t block_token_pg(const AttParams& p, const Item& it, int jb, int32_t pg) {
  const int64_t key = it.kbeg + (int64_t)jb * kBK;
  if constexpr (kPaged)
    return (int64_t)pg * 128 + (key & 127);
  else
    return it.bh * p.Tkv + key;
}

// prefetch the 16-key block at item-relative key k0 of one role into L2
template <int W, int BR, bool kPaged>
__device__ __forceinline__ void prefetch_block(const AttParams& p, const AttView& v, const Item& it,
                                               int k0, bool scales2) {
  const int64_t tok = token_of<kPaged>(p, it, k0);  // 16 keys share one page (k0 % 16 == 0)
  prefetch_l2(v.idxw + tok * W, kBK * W * 4);
  prefetch_l2(v.radw + tok * BR, kBK * BR * 4);
  if (scales2) {
    prefetch_l2(p.k.scales + tok, kBK * 2);
    prefetch_l2(p.v.scales + tok, kBK * 2);
  }
}

// --------------------------------------------------------------- K block
// lane (g4, t4) decodes chunks 8 t4 .. 8 t4 + 7 of keys g4 and g4 + 8
template <int W, int BR>
struct KRegs {
  using Run = IdxRun<8, W, 4>;
  static constexpr int kRW = BR == 4 ? 1 : 2;
  uint32_t ia[Run::kNW], ib[Run::kNW], ra[kRW], rb[kRW];
  __half ska, skb, sva, svb;  // fp16 K and V scales of keys a, b
};
// the block's first token in the streams (16 keys never straddle a page)
template <bool kPaged>
__device__ __forceinline__ int64_t block_token(const AttParams& p, const Item& it, int k0) {
  return token_of<kPaged>(p, it, k0);
}
// per-lane word offsets of a K block (block-relative keys ka, kb)
struct KOffs {
  uint32_t ia, ib, ra, rb, ka, kb;
};
template <int W, int BR>
__device__ __forceinline__ KOffs k_offs(int ka, int kb, int t4) {
  const uint32_t wo = ((uint32_t)t4 * 8u * W) >> 5, ro = ((uint32_t)t4 * 8u * BR) >> 5;
  return KOffs{(uint32_t)ka * W + wo, (uint32_t)kb * W + wo, (uint32_t)ka * BR + ro,
               (uint32_t)kb * BR + ro, (uint32_t)ka, (uint32_t)kb};
}
template <int W, int BR>
__device__ __forceinline__ void k_load(KRegs<W, BR>& r, const AttParams& p, int64_t tok0, const KOffs& o) {
  using R = KRegs<W, BR>;
  const uint32_t* ib = p.k.idxw + tok0 * W;  // warp-uniform block bases
  const uint32_t* rb = p.k.radw + tok0 * BR;
  const __half* ks = reinterpret_cast<const __half*>(p.k.scales) + tok0;
  const __half* vs = reinterpret_cast<const __half*>(p.v.scales) + tok0;
#pragma unroll
  for (int i = 0; i < R::Run::kNW; ++i) {
    r.ia[i] = ib[o.ia + i];
    r.ib[i] = ib[o.ib + i];
  }
#pragma unroll
  for (int i = 0; i < R::kRW; ++i) {
    r.ra[i] = rb[o.ra + i];
    r.rb[i] = rb[o.rb + i];
  }
  r.ska = ks[o.ka];
  r.skb = ks[o.kb];
  r.sva = vs[o.ka];
  r.svb = vs[o.kb];
}

// --------------------------------------------------------------- V block
// lane (g4, t4) decodes chunks 4 g4 .. 4 g4 + 3 of keys 2t4, 2t4+1, 2t4+8, 2t4+9
template <int W, int BR>
struct VRegs {
  using Run = IdxRun<4, W, 8>;
  uint32_t iw[4][Run::kNW];
  uint32_t rw[4][2];
};
// per-lane word offsets of a V block: keys 2t4, 2t4+1, 2t4+8, 2t4+9 (clamped)
struct VOffs {
  uint32_t i[4], r[4];
};
template <int W, int BR>
__device__ __forceinline__ VOffs v_offs(int klast, int g4, int t4) {
  VOffs o;
  const uint32_t wo = ((uint32_t)g4 * 4u * W) >> 5, ro = ((uint32_t)g4 * 4u * BR) >> 5;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int k = min((e >> 1) * 8 + t4 * 2 + (e & 1), klast);
    o.i[e] = (uint32_t)k * W + wo;
    o.r[e] = (uint32_t)k * BR + ro;
  }
  return o;
}
template <int W, int BR>
__device__ __forceinline__ void v_load(VRegs<W, BR>& r, const AttParams& p, int64_t tok0, const VOffs& o,
                                       bool two) {
  using R = VRegs<W, BR>;
  const uint32_t* ib = p.v.idxw + tok0 * W;  // warp-uniform block bases
  const uint32_t* rb = p.v.radw + tok0 * BR;
#pragma unroll
  for (int e = 0; e < 4; ++e) {
#pragma unroll
    for (int i = 0; i < R::Run::kNW; ++i) r.iw[e][i] = ib[o.i[e] + i];
    r.rw[e][0] = rb[o.r[e]];
    r.rw[e][1] = two ? rb[o.r[e] + 1] : 0u;
  }
}

// ----------------------------------------------------------------- kernel
template <int W, int BR, bool kPaged>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kCThreads, 1)
    attention_pair_kernel(const CParams c) {
  extern __shared__ __align__(128) unsigned char sm[];
  const AttParams& p = c.p;
  const uint32_t role = cta_rank();  // 0: K CTA, 1: V CTA
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g4 = lane >> 2, t4 = lane & 3;
  uint2* tab = reinterpret_cast<uint2*>(sm);
  unsigned char* mslot = sm + kBoxOff + warp * kWarpMsg;  // this warp's mailbox (V CTA)
  uint64_t* mbox = reinterpret_cast<uint64_t*>(sm + kBarOff) + warp;
  const uint32_t peer = role ^ 1u;

  const int nclus = gridDim.x / 2;
  const int64_t clus = blockIdx.x / 2;
  const int64_t i0 = (int64_t)((uint64_t)clus * (uint64_t)c.items / (uint32_t)nclus);
  const int64_t i1 = (int64_t)((uint64_t)(clus + 1) * (uint64_t)c.items / (uint32_t)nclus);

  if (lane == 0) {
    mbar_init(mbox, 1);
    fence_mbar_init();
    if (role == 1) mbar_arrive_expect_tx(mbox, kWarpMsg);  // phase 0 expects the first message
  }
  __syncthreads();
  cluster_sync();  // the peer's barriers are initialised before any remote op
  const uint32_t mbox_peer = mapa(smem_u32(mbox), peer);
  const uint32_t mslot_peer = mapa(smem_u32(mslot), peer);
  const uint32_t tab_lane = smem_u32(tab) + (uint32_t)(lane & 15) * 8u;  // this lane's replica
  const AttView& own = role == 0 ? p.k : p.v;
  uint32_t u = 0;  // mailbox uses of this warp
  int64_t cur_hkv = -1;

  for (int64_t ii = i0; ii < i1; ++ii) {
    const Item it = item_at(c, ii);
    if (it.hkv != cur_hkv) {  // (re)load this role's replicated table
      __syncthreads();
      fill_table(tab, own.table16 + it.hkv * c.ncw, c.ncw, tid);
      __syncthreads();
      cur_hkv = it.hkv;
    }
    const int64_t row_stride = (int64_t)c.nsplit * kCW;
    const int64_t part = (it.bh * p.nrows) * row_stride + (int64_t)it.split * kCW + warp;
    if (kPfDist > 0 && lane == 0)
      for (int d = 0; d < kPfDist; ++d) {
        const int j = warp + d * kCW;
        if (j < it.nblk) prefetch_block<W, BR, kPaged>(p, own, it, j * kBK, role == 0);
      }
    if (role == 0) {
      // ======================================================== K warp
      // S^T = K Q^T: A = the decoded keys (rows g4, g4 + 8 of the M = 16
      // block), B = Q^T (N = 8 query rows), 16 permuted dims per k-slab:
      // lane t4's dims of slab ks are the 4 components of chunk 8 t4 + ks.
      using R = KRegs<W, BR>;
      uint32_t qb[8][2];
      {
        // softmax scale * log2(e) * 2^9 / top (the decoded products are q c 2^-9)
        const float qs = c.q_scale;
        const bool rv = g4 < p.nrows;
        const int gi = rv ? g4 / (int)p.Tq : 0, qi = rv ? g4 - gi * (int)p.Tq : 0;
        const float4* qrow = reinterpret_cast<const float4*>(
            p.q + ((it.b * p.Hq + it.hkv * p.g + gi) * p.Tq + qi) * 128);
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
          if (rv) v = __ldg(qrow + 8 * t4 + ks);
          qb[ks][0] = pack_half2(v.x * qs, v.y * qs);
          qb[ks][1] = pack_half2(v.z * qs, v.w * qs);
        }
      }
      const int64_t tkv = p.kv_lens ? (int64_t)__ldg(p.kv_lens + it.b) : p.Tkv;
      // rows r0 = 2 t4, r1 = 2 t4 + 1 of this lane; keys visible to them and to
      // every row (item-relative).  Rows >= nrows carry zero queries: their
      // values stay finite and are never written.
      const int r0 = 2 * t4, r1 = 2 * t4 + 1;
      int vis0 = it.kend_rel, vis1 = it.kend_rel, vis_min = it.kend_rel;
      if (p.causal) {
        const int64_t off = tkv - p.Tq + 1 - it.kbeg;
        auto clampv = [&](int64_t v) { return (int)max((int64_t)0, min((int64_t)it.kend_rel, v)); };
        vis0 = clampv((r0 % (int)p.Tq) + off);
        vis1 = clampv((r1 % (int)p.Tq) + off);
        vis_min = clampv(off);
      }
      const uint32_t sh_i = ((uint32_t)t4 * 8u * W) & 31u, sh_r = ((uint32_t)t4 * 8u * BR) & 31u;
      // running maxima start at a finite floor so that fully masked rows give
      // p = 2^-inf = 0 without special cases
      float m0 = -1e30f, m1 = -1e30f, l0 = 0.f, l1 = 0.f;  // l: this lane's partial sums
      const KOffs ko_full = k_offs<W, BR>(g4, g4 + 8, t4);
      auto kload = [&](R& r, int jb, int32_t pg) {
        const int k0 = jb * kBK, klast = it.kend_rel - 1 - k0;
        int64_t tok;
        if constexpr (kPaged) tok = block_token_pg<true>(p, it, jb, pg);
        else tok = block_token<false>(p, it, k0);
        if (klast >= kBK - 1)
          k_load<W, BR>(r, p, tok, ko_full);
        else  // the item's partial last block: clamp to its last key
          k_load<W, BR>(r, p, tok, k_offs<W, BR>(min(g4, klast), min(g4 + 8, klast), t4));
      };
      R nx;
      if (warp < it.nblk) kload(nx, warp, kPaged ? block_page<kPaged>(p, it, warp) : 0);
      int32_t pg_next = 0;  // (paged: the page of the block loaded next)
      if constexpr (kPaged)
        if (warp + kCW < it.nblk) pg_next = block_page<true>(p, it, warp + kCW);
      for (int j = warp; j < it.nblk; j += kCW) {
        // everything this block needs is taken out of the load buffer first,
        // then the next block is loaded into the same registers (no copies)
        if (kPfDist > 0 && lane == 0 && j + kPfDist * kCW < it.nblk)
          prefetch_block<W, BR, kPaged>(p, own, it, (j + kPfDist * kCW) * kBK, true);
        typename R::Run ia, ib;
        ia.align(nx.ia, sh_i);
        ib.align(nx.ib, sh_i);
        const float2 sk = __half22float2(__halves2half2(nx.ska, nx.skb));
        float2 sv = __half22float2(__halves2half2(nx.sva, nx.svb));
        uint32_t rq[4];  // radius words: b_r 4 -> (ra0, ra1, rb0, rb1); else (ra, rb, ra2, rb2)
        if constexpr (BR == 4) {
          rq[0] = nx.ra[0];
          rq[1] = rq[0] >> 4;
          rq[2] = nx.rb[0];
          rq[3] = rq[2] >> 4;
        } else {
          rq[0] = __funnelshift_r(nx.ra[0], nx.ra[1], sh_r);
          rq[1] = __funnelshift_r(nx.rb[0], nx.rb[1], sh_r);
          rq[2] = nx.ra[1] >> sh_r;
          rq[3] = nx.rb[1] >> sh_r;
        }
        if (j + kCW < it.nblk) {
          kload(nx, j + kCW, pg_next);
          if constexpr (kPaged)
            if (j + 2 * kCW < it.nblk) pg_next = block_page<true>(p, it, j + 2 * kCW);
        }
        float sc[4] = {0.f, 0.f, 0.f, 0.f};
        if constexpr (BR == 4) {
          const uint32_t ra0 = rq[0], ra1 = rq[1], rb0 = rq[2], rb1 = rq[3];
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const uint2 ca = lds64(ia.addr(ks, tab_lane));
            const uint2 cb = lds64(ib.addr(ks, tab_lane));
            uint32_t qa_, qb_;
            switch (ks) {
              case 0: qa_ = rad4<0>(ra0); qb_ = rad4<0>(rb0); break;
              case 1: qa_ = rad4<0>(ra1); qb_ = rad4<0>(rb1); break;
              case 2: qa_ = rad4<1>(ra0); qb_ = rad4<1>(rb0); break;
              case 3: qa_ = rad4<1>(ra1); qb_ = rad4<1>(rb1); break;
              case 4: qa_ = rad4<2>(ra0); qb_ = rad4<2>(rb0); break;
              case 5: qa_ = rad4<2>(ra1); qb_ = rad4<2>(rb1); break;
              case 6: qa_ = rad4<3>(ra0); qb_ = rad4<3>(rb0); break;
              default: qa_ = rad4<3>(ra1); qb_ = rad4<3>(rb1); break;
            }
            mma_f(sc, hmul2_raw(qa_, ca.x), hmul2_raw(qb_, cb.x), hmul2_raw(qa_, ca.y),
                  hmul2_raw(qb_, cb.y), qb[ks][0], qb[ks][1]);
          }
        } else {
          const uint32_t ra = rq[0], rb = rq[1], ra2 = rq[2], rb2 = rq[3];
          constexpr uint32_t kRM = (1u << BR) - 1u;
#pragma unroll
          for (int ks = 0; ks < 8; ++ks) {
            const uint2 ca = lds64(ia.addr(ks, tab_lane));
            const uint2 cb = lds64(ib.addr(ks, tab_lane));
            uint32_t qa_, qb_;
            if (ks * BR + BR <= 32) {
              qa_ = radq((ra >> (ks * BR)) & kRM);
              qb_ = radq((rb >> (ks * BR)) & kRM);
            } else if (ks * BR < 32) {  // a code straddling the aligned run's first word
              qa_ = radq(__funnelshift_r(ra, ra2, ks * BR) & kRM);
              qb_ = radq(__funnelshift_r(rb, rb2, ks * BR) & kRM);
            } else {
              qa_ = radq((ra2 >> (ks * BR - 32)) & kRM);
              qb_ = radq((rb2 >> (ks * BR - 32)) & kRM);
            }
            mma_f(sc, hmul2_raw(qa_, ca.x), hmul2_raw(qb_, cb.x), hmul2_raw(qa_, ca.y),
                  hmul2_raw(qb_, cb.y), qb[ks][0], qb[ks][1]);
          }
        }
        // sc = S^T[key a][r0], [a][r1], [b][r0], [b][r1]; per-key sigma_k
        float s00 = sc[0] * sk.x, s01 = sc[1] * sk.x, s10 = sc[2] * sk.y, s11 = sc[3] * sk.y;
        const int kt0 = j * kBK;
        if (kt0 + kBK > vis_min) {  // some key of this block is masked (warp-uniform)
          const int ka = kt0 + g4, kb = ka + 8;
          if (ka >= vis0) s00 = -INFINITY;
          if (ka >= vis1) s01 = -INFINITY;
          if (kb >= vis0) s10 = -INFINITY;
          if (kb >= vis1) s11 = -INFINITY;
          if (ka >= it.kend_rel) sv.x = 0.f;
          if (kb >= it.kend_rel) sv.y = 0.f;
        }
        // block max of rows r0, r1 over the 16 keys (lanes g4)
        float x0 = fmaxf(s00, s10), x1 = fmaxf(s01, s11);
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, o));
          x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, o));
        }
        // lazy running max: raised only when the block exceeds it by > kLazy
        // (P stays <= 2^8 in fp16 and most blocks need no rescale)
        float a0 = 1.f, a1 = 1.f;
        if (x0 > m0 + kLazy) {
          a0 = ex2(m0 - x0);
          m0 = x0;
        }
        if (x1 > m1 + kLazy) {
          a1 = ex2(m1 - x1);
          m1 = x1;
        }
        const float p00 = ex2(s00 - m0), p10 = ex2(s10 - m0);
        const float p01 = ex2(s01 - m1), p11 = ex2(s11 - m1);
        l0 = l0 * a0 + (p00 + p10);
        l1 = l1 * a1 + (p01 + p11);
        // P (with sigma_v; 2^9 / top is applied by the combine) to the V twin
        const uint32_t w0 = pack_half2(p00 * sv.x, p10 * sv.y);  // row r0: keys a, b
        const uint32_t w1 = pack_half2(p01 * sv.x, p11 * sv.y);  // row r1
        mbar_wait(mbox, (u & 1u) ^ 1u);  // the V twin has consumed the previous message
        st_async4(mslot_peer + r0 * 32u + g4 * 4u, mbox_peer, w0);
        st_async4(mslot_peer + r1 * 32u + g4 * 4u, mbox_peer, w1);
        if (g4 == 0) st_async8(mslot_peer + kMsgP + r0 * 4u, mbox_peer, __float_as_uint(a0), __float_as_uint(a1));
        ++u;
      }
      // row sums over the lanes g4
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        l0 += __shfl_xor_sync(0xffffffffu, l0, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
      }
      if (g4 == 0) {
        if (r0 < p.nrows) {
          const int64_t idx = part + r0 * row_stride;
          p.part_ml[2 * idx] = m0;
          p.part_ml[2 * idx + 1] = l0;
        }
        if (r1 < p.nrows) {
          const int64_t idx = part + r1 * row_stride;
          p.part_ml[2 * idx] = m1;
          p.part_ml[2 * idx + 1] = l1;
        }
      }
    } else {
      // ======================================================== V warp
      using R = VRegs<W, BR>;
      float oT[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) oT[i][0] = oT[i][1] = oT[i][2] = oT[i][3] = 0.f;
      const uint32_t sh_i = ((uint32_t)g4 * 4u * W) & 31u, sh_r = ((uint32_t)g4 * 4u * BR) & 31u;
      const bool two = BR * 4 + (((uint32_t)g4 * 4u * BR) & 31u) > 32u;  // radius run spans 2 words
      const VOffs vo_full = v_offs<W, BR>(kBK - 1, g4, t4);
      auto vload = [&](R& r, int jb, int32_t pg) {
        const int k0 = jb * kBK, klast = it.kend_rel - 1 - k0;
        int64_t tok;
        if constexpr (kPaged) tok = block_token_pg<true>(p, it, jb, pg);
        else tok = block_token<false>(p, it, k0);
        if (klast >= kBK - 1)
          v_load<W, BR>(r, p, tok, vo_full, two);
        else
          v_load<W, BR>(r, p, tok, v_offs<W, BR>(klast, g4, t4), two);
      };
      R nx;
      if (warp < it.nblk) vload(nx, warp, kPaged ? block_page<kPaged>(p, it, warp) : 0);
      int32_t pg_next = 0;  // (paged: the page of the block loaded next)
      if constexpr (kPaged)
        if (warp + kCW < it.nblk) pg_next = block_page<true>(p, it, warp + kCW);
      for (int j = warp; j < it.nblk; j += kCW) {
        if (kPfDist > 0 && lane == 0 && j + kPfDist * kCW < it.nblk)
          prefetch_block<W, BR, kPaged>(p, own, it, (j + kPfDist * kCW) * kBK, false);
        typename R::Run ic[4];
        uint32_t rr[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          ic[e].align(nx.iw[e], sh_i);
          rr[e] = __funnelshift_r(nx.rw[e][0], nx.rw[e][1], sh_r);  // 4 codes of this lane
        }
        if (j + kCW < it.nblk) {  // (into the registers just consumed)
          vload(nx, j + kCW, pg_next);
          if constexpr (kPaged)
            if (j + 2 * kCW < it.nblk) pg_next = block_page<true>(p, it, j + 2 * kCW);
        }
        mbar_wait(mbox, u & 1u);  // the K twin's message has landed (complete-tx)
        // P^T B fragment of row g4, keys 2t4, 2t4+1, 2t4+8, 2t4+9 (positions
        // 4 t4 .. 4 t4 + 3 hold keys 2t4, 2t4+8, 2t4+1, 2t4+9); rescale
        // factors of rows 2 t4, 2 t4 + 1 (this lane's O^T columns)
        const uint2 pw = *reinterpret_cast<const uint2*>(mslot + g4 * 32 + t4 * 8);
        const float2 al = *reinterpret_cast<const float2*>(mslot + kMsgP + t4 * 8);
        // the mailbox is overwritten once freed: complete the loads (their
        // registers are inputs here) before the relaxed remote arrive
        asm volatile("" ::"r"(pw.x), "r"(pw.y), "f"(al.x), "f"(al.y) : "memory");
        __syncwarp();
        if (lane == 0) {
          mbar_arrive_expect_tx(mbox, kWarpMsg);  // re-arm for the next message
          remote_arrive(mbox_peer);               // mailbox free for the K twin
        }
        ++u;
        const uint32_t pb0 = __byte_perm(pw.x, pw.y, 0x5410), pb1 = __byte_perm(pw.x, pw.y, 0x7632);
        if (__any_sync(0xffffffffu, al.x != 1.f || al.y != 1.f)) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            oT[i][0] *= al.x; oT[i][1] *= al.y; oT[i][2] *= al.x; oT[i][3] *= al.y;
          }
        }
#pragma unroll
        for (int jj = 0; jj < 4; ++jj) {
          uint2 vv[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const uint2 cw = lds64(ic[e].addr(jj, tab_lane));
            uint32_t qq;
            if constexpr (BR == 4)
              qq = (jj == 0 ? rad4<0>(rr[e]) : jj == 1 ? rad4<0>(rr[e] >> 4)
                    : jj == 2 ? rad4<1>(rr[e]) : rad4<1>(rr[e] >> 4));
            else
              qq = radq((rr[e] >> (jj * BR)) & ((1u << BR) - 1u));
            vv[e] = make_uint2(hmul2_raw(qq, cw.x), hmul2_raw(qq, cw.y));
          }
          // m-tile 2jj: (m = g4, g4+8) = elements (0, 1); m-tile 2jj+1: elements (2, 3)
          mma_f(oT[2 * jj], __byte_perm(vv[0].x, vv[1].x, 0x5410), __byte_perm(vv[0].x, vv[1].x, 0x7632),
                __byte_perm(vv[2].x, vv[3].x, 0x5410), __byte_perm(vv[2].x, vv[3].x, 0x7632), pb0, pb1);
          mma_f(oT[2 * jj + 1], __byte_perm(vv[0].y, vv[1].y, 0x5410), __byte_perm(vv[0].y, vv[1].y, 0x7632),
                __byte_perm(vv[2].y, vv[3].y, 0x5410), __byte_perm(vv[2].y, vv[3].y, 0x7632), pb0, pb1);
        }
      }
      // this warp's partial O^T: element (mt, e) = (dim, row)
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int row = t4 * 2 + (e & 1);
          const int dim = 4 * (4 * g4 + (mt >> 1)) + 2 * (mt & 1) + (e >> 1);
          if (row < p.nrows) p.part_o[(part + row * row_stride) * 128 + dim] = oT[mt][e];
        }
      }
    }
  }
  __syncwarp();
  cluster_sync();  // no CTA leaves while its peer may still address its shared memory
}

template <int W, int BR, bool kPaged>
int launch_pair(const CParams& c, cudaStream_t st) {
  auto kern = attention_pair_kernel<W, BR, kPaged>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
  if (e != cudaSuccess) return record_cuda_error(e);
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(kCThreads);
  cfg.dynamicSmemBytes = kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 2;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  int nclus = 0;
  cfg.gridDim = dim3(2 * kNcMax);
  e = cudaOccupancyMaxActiveClusters(&nclus, kern, &cfg);
  if (e != cudaSuccess || nclus < 1) nclus = kNcMax / 2;
  nclus = (int)std::min<int64_t>({(int64_t)nclus, (int64_t)kNcMax, c.items});
  cfg.gridDim = dim3(2 * nclus);
  e = cudaLaunchKernelEx(&cfg, kern, c);
  return e == cudaSuccess ? HQMQ_OK : record_cuda_error(e);
}

template <bool kPaged>
int dispatch_pair(const CParams& c, int w, int br, cudaStream_t st) {
  switch (w * 16 + br) {
    case 9 * 16 + 4: return launch_pair<9, 4, kPaged>(c, st);     // S = 16
    case 10 * 16 + 4: return launch_pair<10, 4, kPaged>(c, st);
    case 11 * 16 + 4: return launch_pair<11, 4, kPaged>(c, st);   // S = 43..64
    case 11 * 16 + 6: return launch_pair<11, 6, kPaged>(c, st);   // Qwen config b_r 6
    case 11 * 16 + 3: return launch_pair<11, 3, kPaged>(c, st);
    default: return HQMQ_ERR_UNSUPPORTED;
  }
}

}  // namespace

// Split plan shared by the workspace query and the launch: ~4 items per
// cluster, splits aligned to 128 keys (pages).
void pair_plan(int64_t rows, int64_t tkv, int& nsplit, int64_t& kps) {
  const int64_t ntile = std::max<int64_t>(1, ceil_div(tkv, 128));
  int64_t s = std::min<int64_t>(ntile, std::max<int64_t>(1, ceil_div(4 * kNcMax, rows)));
  kps = ceil_div(ntile, s) * 128;
  nsplit = (int)ceil_div(tkv, kps);
}

bool pair_applicable(int64_t bhkv, int64_t head_dim, int64_t nrows, int64_t tkv, int S, int w, int br,
                     bool flags, const void* t16k, const void* t16v) {
  if (head_dim != 128 || flags || nrows > 8 || tkv < 1 || !t16k || !t16v) return false;
  // each CTA replicates its table into 192 KB of shared memory: worth it from
  // ~4M cached keys (B = 32 x 8 heads x 16k); smaller caches keep the
  // single-CTA kernel (measured: B=1 x 8 x 32k 0.047 vs 0.134 ms)
  if (bhkv * tkv < (int64_t(1) << 22)) return false;
  if ((int64_t)kGroupOrder * S > kMaxCw) return false;
  switch (w * 16 + br) {
    case 9 * 16 + 4: case 10 * 16 + 4: case 11 * 16 + 4: case 11 * 16 + 6: case 11 * 16 + 3:
      return true;
    default:
      return false;
  }
}

size_t pair_workspace(int64_t bhkv, int64_t nrows, int64_t tkv) {
  int nsplit;
  int64_t kps;
  pair_plan(bhkv, tkv, nsplit, kps);
  return (size_t)bhkv * nrows * nsplit * kCW * (128 + 2) * sizeof(float) + 256;
}

// p: parameters as for attention_mma_kernel; p.part_o points at a workspace
// of pair_workspace bytes.  Launches the pair kernel and the combine.
int launch_pair_attention(AttParams p, int64_t max_tkv, cudaStream_t st) {
  CParams c;
  pair_plan(p.B * p.Hkv, max_tkv, c.nsplit, c.kps);
  c.items = p.Hkv * p.B * c.nsplit;
  if (c.items >= (1ll << 31)) return HQMQ_ERR_UNSUPPORTED;
  c.ncw = kGroupOrder * p.S;
  c.q_scale = p.scale_log2 * kProdScale / (float)((1 << p.br) - 1);
  const int64_t parts = p.B * p.Hkv * p.nrows * c.nsplit * kCW;
  p.part_ml = p.part_o + parts * 128;
  c.p = p;
  const int rc = p.kv_lens ? dispatch_pair<true>(c, p.w, p.br, st) : dispatch_pair<false>(c, p.w, p.br, st);
  if (rc != HQMQ_OK) return rc;
  AttParams q = p;
  q.splits = c.nsplit * kCW;
  q.o_scale = kProdScale / (float)((1 << p.br) - 1);  // the decoded V products are q c 2^-9
  combine_kernel<<<dim3((unsigned)(p.B * p.Hkv), (unsigned)p.nrows), 128, 0, st>>>(q);
  return check_launch();
}

}  // namespace hqmq
