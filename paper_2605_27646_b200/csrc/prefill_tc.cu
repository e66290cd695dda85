// Prefill attention on the 5th-gen tensor cores (the
// paper's weakest number).  Prefill reads every key many
// times (once per 128-row query tile), so the compressed K / V are decoded
// ONCE into an fp16 workspace by the HBM-bound decode kernels and this kernel
// runs flash attention over them:
//
//   CTA = 128 query rows ((128 / g) query tokens x the g query heads of one
//   kv head) = 4 warps = the 128 TMEM lanes; per 64-key tile
//     K tile -> smem (UMMA K-major canonical layout), S = Q K^T:
//       tcgen05.mma kind::f16, M=128, N=64, 8 x K=16 steps, fp32 S in TMEM
//     each thread owns one row: tcgen05.ld its 64 scores, causal mask,
//       online softmax in the log2 domain, O (fp32, TMEM) rescaled in place
//       (tcgen05.ld / st) when the row max grows, P -> smem fp16 (K-major)
//     V tile -> smem (MN-major: rows of V are already dim-contiguous),
//       O += P V: M=128, N=128, 4 x K=16 steps into the TMEM accumulator
//   descriptors SWIZZLE_NONE, one thread issues, tcgen05.commit -> mbarrier.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "common.cuh"

namespace hqmq {

constexpr int kFaRows = 128, kFaKeys = 64, kFaD = 128, kFaThreads = 128;
// canonical layouts: core matrix = 8 rows x 16 bytes
//   K-major (Q, K, P): byte(r, k) = (r/8)*SBO + (k/8)*128 + (r%8)*16 + (k%8)*2
//   MN-major (V):      byte(n, k) = (n/8)*SBO + (k/8)*128 + (k%8)*16 + (n%8)*2
constexpr uint32_t kFaLBO = 128;
constexpr uint32_t kSboQK = (kFaD / 8) * 128;    // 16 k-groups per 8-row group: 2048
constexpr uint32_t kSboP = (kFaKeys / 8) * 128;  // 8 k-groups: 1024
constexpr uint32_t kSboV = (kFaKeys / 8) * 128;  // 8 key-groups per 8-dim group: 1024
constexpr uint32_t kQBytes = kFaRows * kFaD * 2, kKBytes = kFaKeys * kFaD * 2;

__device__ __forceinline__ uint64_t fa_desc(uint32_t saddr, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)(kFaLBO >> 4) << 16) |
         ((uint64_t)(sbo >> 4) << 32) | ((uint64_t)1 << 46);
}
__host__ __device__ constexpr uint32_t fa_idesc(int M, int N, int b_mn_major) {
  return (1u << 4) | ((uint32_t)b_mn_major << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void fa_mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void fa_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
      smem_u32(bar)));
}
#define FA_LD32(addr, r)                                                                        \
  asm volatile(                                                                                 \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"      \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),   \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),              \
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),           \
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),           \
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),           \
        "=r"(r[31])                                                                             \
      : "r"(addr))
#define FA_ST32(addr, r)                                                                        \
  asm volatile(                                                                                 \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12," \
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"     \
      ::"r"(addr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), \
        "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]),         \
        "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]),      \
        "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),      \
        "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]))

struct FaParams {
  int64_t B, Hq, Hkv, Tq, Tkv;
  int g, causal;
  float scale_log2;
  const float* q;     // (B, Hq, Tq, 128) fp32
  const __half* k;    // (B, Hkv, Tkv, 128) fp16 (decoded)
  const __half* v;
  float* out;         // (B, Hq, Tq, 128) fp32
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 16 : 0)
               : "memory");
}

__global__ void __launch_bounds__(kFaThreads, 2) attention_fa_tc_kernel(FaParams p) {
  extern __shared__ __align__(1024) unsigned char fsm[];
  unsigned char* qs = fsm;                       // 32 KB
  unsigned char* kvbuf = qs + kQBytes;           // 2 x (K 16 KB + V 16 KB): cp.async double buffer
  unsigned char* psm = kvbuf + 4 * kKBytes;      // 16 KB (P)
  __shared__ __align__(8) uint64_t bar_s, bar_o;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int64_t bh = blockIdx.y;
  const int64_t b = bh / p.Hkv, hkv = bh % p.Hkv;
  const int g = p.g;
  const int tpt = kFaRows / g;
  const int64_t tok0 = (int64_t)blockIdx.x * tpt;
  const int64_t off = p.causal ? (p.Tkv - p.Tq) : 0;
  // this thread's row
  const int64_t qtok = tok0 + tid / g;
  const int qhead = tid % g;
  const bool rvalid = qtok < p.Tq;
  const int64_t vis = p.causal ? qtok + off + 1 : p.Tkv;

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&bar_s, 1);
    mbar_init(&bar_o, 1);
    fence_mbar_init();
  }
  // Q row -> fp16 (pre-scaled), K-major A operand
  {
    const float4* qr = reinterpret_cast<const float4*>(
        p.q + ((b * p.Hq + hkv * g + qhead) * p.Tq + (rvalid ? qtok : 0)) * kFaD);
#pragma unroll 4
    for (int kg = 0; kg < kFaD / 8; ++kg) {
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f), c = a;
      if (rvalid) {
        a = __ldg(qr + 2 * kg);
        c = __ldg(qr + 2 * kg + 1);
      }
      const float sl = p.scale_log2;
      const __half2 h0 = __floats2half2_rn(a.x * sl, a.y * sl), h1 = __floats2half2_rn(a.z * sl, a.w * sl);
      const __half2 h2 = __floats2half2_rn(c.x * sl, c.y * sl), h3 = __floats2half2_rn(c.z * sl, c.w * sl);
      *reinterpret_cast<uint4*>(qs + (tid >> 3) * kSboQK + kg * 128 + (tid & 7) * 16) =
          make_uint4(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1),
                     *reinterpret_cast<const uint32_t*>(&h2), *reinterpret_cast<const uint32_t*>(&h3));
    }
  }
  fence_proxy_async();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_slot;  // S(t & 1): cols [0, 64) / [64, 128), O: cols [128, 256)
  const uint32_t tm_row = tm + ((uint32_t)(warp * 32) << 16);
  const uint32_t q_sa = smem_u32(qs), p_sa = smem_u32(psm);

  const int64_t last_tok = std::min(p.Tq, tok0 + tpt) - 1;
  const int64_t kend = p.causal ? std::min(p.Tkv, last_tok + off + 1) : p.Tkv;
  const __half* kbase = p.k + bh * p.Tkv * kFaD;
  const __half* vbase = p.v + bh * p.Tkv * kFaD;
  float m_run = -INFINITY, l_run = 0.f;
  uint32_t ph_s = 0, ph_o = 0;
  const int ntiles = (int)((kend + kFaKeys - 1) / kFaKeys);
  // K tiles run two ahead (K-major B: row = key), V tiles one ahead (MN-major
  // B: n = dim, k = key), each double-buffered and zero-filled past kend; every
  // call commits one cp.async group so the group count stays uniform
  auto load_k = [&](int t) {
    if (t < ntiles) {
      unsigned char* ks = kvbuf + (t & 1) * kKBytes;
      const int64_t k0 = (int64_t)t * kFaKeys;
      for (int i = tid; i < kFaKeys * (kFaD / 8); i += kFaThreads) {
        const int key = i >> 4, dg = i & 15;
        const bool ok = k0 + key < kend;
        cp_async16(ks + (key >> 3) * kSboQK + dg * 128 + (key & 7) * 16,
                   reinterpret_cast<const uint4*>(kbase + (ok ? k0 + key : 0) * kFaD) + dg, ok);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  auto load_v = [&](int t) {
    if (t < ntiles) {
      unsigned char* vs = kvbuf + (2 + (t & 1)) * kKBytes;
      const int64_t k0 = (int64_t)t * kFaKeys;
      for (int i = tid; i < kFaKeys * (kFaD / 8); i += kFaThreads) {
        const int key = i >> 4, dg = i & 15;
        const bool ok = k0 + key < kend;
        cp_async16(vs + dg * kSboV + (key >> 3) * 128 + (key & 7) * 16,
                   reinterpret_cast<const uint4*>(vbase + (ok ? k0 + key : 0) * kFaD) + dg, ok);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  const uint32_t kv_sa = smem_u32(kvbuf);
  auto issue_s = [&](int t) {  // S(t) = Q K(t)^T into TMEM columns (t & 1) * 64
#pragma unroll
    for (int kk = 0; kk < kFaD / 16; ++kk)
      fa_mma(tm + (uint32_t)(t & 1) * 64, fa_desc(q_sa + kk * 256, kSboQK),
             fa_desc(kv_sa + (t & 1) * kKBytes + kk * 256, kSboQK), fa_idesc(kFaRows, kFaKeys, 0),
             kk > 0);
    fa_commit(&bar_s);
  };
  if (ntiles > 0) {
    load_k(0);
    load_k(1);
    load_v(0);
    asm volatile("cp.async.wait_group 2;" ::: "memory");
    fence_proxy_async();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      issue_s(0);
    }
  }
  for (int t = 0; t < ntiles; ++t) {
    const int64_t k0 = (int64_t)t * kFaKeys;
    const int nk = (int)std::min((int64_t)kFaKeys, kend - k0);
    // 1. scores of tile t
    mbar_wait(&bar_s, ph_s);
    ph_s ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t sr[64];
    FA_LD32(tm_row + (uint32_t)(t & 1) * 64, sr);
    FA_LD32(tm_row + (uint32_t)(t & 1) * 64 + 32, (sr + 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    // 2. K(t) is consumed: its buffer takes K(t+2)
    load_k(t + 2);
    // 3. online softmax (log2 domain), P in registers
    float mx = -INFINITY;
#pragma unroll
    for (int j = 0; j < 64; ++j) {
      const int64_t key = k0 + j;
      float sv = __uint_as_float(sr[j]);
      sv = (rvalid && j < nk && key < vis) ? sv : -INFINITY;
      sr[j] = __float_as_uint(sv);
      mx = fmaxf(mx, sv);
    }
    const float m_new = fmaxf(m_run, mx);
    const float alpha = (m_new == -INFINITY) ? 1.f : exp2f(m_run - m_new);
    float psum = 0.f;
    uint32_t hw[32];
#pragma unroll
    for (int e = 0; e < 32; ++e) {
      const float s0 = __uint_as_float(sr[2 * e]), s1 = __uint_as_float(sr[2 * e + 1]);
      const float e0 = m_new == -INFINITY ? 0.f : exp2f(s0 - m_new);
      const float e1 = m_new == -INFINITY ? 0.f : exp2f(s1 - m_new);
      psum += e0 + e1;
      const __half2 h = __floats2half2_rn(e0, e1);
      hw[e] = *reinterpret_cast<const uint32_t*>(&h);
    }
    l_run = l_run * alpha + psum;
    m_run = m_new;
    // 4. PV(t-1) done: P smem, V buffer (t-1) & 1 and the O accumulator are free
    if (t > 0) {
      mbar_wait(&bar_o, ph_o);
      ph_o ^= 1u;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    // 5. V(t+1) into the freed V buffer
    load_v(t + 1);
    // 6. rescale O in TMEM when some row's max moved (warp-uniform), write P(t)
    if (t > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t orr[32];
        FA_LD32(tm_row + 128 + c * 32, orr);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int j = 0; j < 32; ++j) orr[j] = __float_as_uint(__uint_as_float(orr[j]) * alpha);
        FA_ST32(tm_row + 128 + c * 32, orr);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
#pragma unroll
    for (int kg = 0; kg < 8; ++kg)
      *reinterpret_cast<uint4*>(psm + (tid >> 3) * kSboP + kg * 128 + (tid & 7) * 16) =
          make_uint4(hw[4 * kg], hw[4 * kg + 1], hw[4 * kg + 2], hw[4 * kg + 3]);
    // 7. K(t+1) and V(t) have landed (the two newest groups may still fly)
    asm volatile("cp.async.wait_group 2;" ::: "memory");
    fence_proxy_async();
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    // 8. O += P(t) V(t); then S(t+1)
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
      for (int kk = 0; kk < kFaKeys / 16; ++kk)
        fa_mma(tm + 128, fa_desc(p_sa + kk * 256, kSboP),
               fa_desc(kv_sa + (2 + (t & 1)) * kKBytes + kk * 256, kSboV),
               fa_idesc(kFaRows, kFaD, 1), (t > 0 || kk > 0) ? 1u : 0u);
      fa_commit(&bar_o);
      if (t + 1 < ntiles) issue_s(t + 1);
    }
  }
  const int ntile = ntiles;
  if (ntile > 0) {
    mbar_wait(&bar_o, ph_o);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  // ---- O / l -> out (every thread takes part in the aligned TMEM loads)
  {
    float* orow = p.out + ((b * p.Hq + hkv * g + qhead) * p.Tq + (rvalid ? qtok : 0)) * kFaD;
    const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t orr[32];
      if (ntile > 0) {
        FA_LD32(tm_row + 128 + c * 32, orr);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) orr[j] = 0u;
      }
      if (rvalid) {
#pragma unroll
        for (int j = 0; j < 32; j += 4)
          *reinterpret_cast<float4*>(orow + c * 32 + j) =
              make_float4(__uint_as_float(orr[j]) * inv, __uint_as_float(orr[j + 1]) * inv,
                          __uint_as_float(orr[j + 2]) * inv, __uint_as_float(orr[j + 3]) * inv);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(256));
}

// Decode-once + tcgen05 flash attention for prefill shapes.  Workspace: the
// two decoded fp16 tensors (kv layout) + an error word.
size_t prefill_tc_workspace(const hqmq_attention_args* a) {
  return 2 * (size_t)a->batch * a->kv_heads * a->kv_tokens * kFaD * 2 + 256;
}

bool prefill_tc_applicable(const hqmq_attention_args* a) {
  if (a->head_dim != kFaD || a->precise) return false;
  const int64_t g = a->q_heads / a->kv_heads;
  return g >= 1 && kFaRows % g == 0 && g * a->q_tokens > 8;
}

int launch_prefill_tc(const hqmq_attention_args* a, cudaStream_t st) {
  unsigned char* ws = reinterpret_cast<unsigned char*>(a->workspace);
  const size_t nelem = (size_t)a->batch * a->kv_heads * a->kv_tokens * kFaD;
  __half* kd = reinterpret_cast<__half*>(ws);
  __half* vd = kd + nelem;
  uint32_t* err = reinterpret_cast<uint32_t*>(ws + 2 * nelem * 2);
  cudaError_t e = cudaMemsetAsync(err, 0, 4, st);
  if (e != cudaSuccess) return record_cuda_error(e);
  for (int t = 0; t < 2; ++t) {
    const hqmq_packed_view& v = t == 0 ? a->k : a->v;
    hqmq_decode_args d{};
    d.batch = a->batch; d.heads = a->kv_heads; d.tokens = a->kv_tokens; d.head_dim = a->head_dim;
    d.codebook_size = a->codebook_size; d.radius_bits = a->radius_bits; d.index_bits = a->index_bits;
    d.out_dtype = HQMQ_F16;
    d.token_start = 0; d.token_stop = a->kv_tokens;
    d.scales = v.scales; d.index_words = v.index_words; d.radius_words = v.radius_words;
    d.flag_words = v.flag_words; d.payloads = v.payloads; d.token_offsets = v.token_offsets;
    d.joint_f32 = v.joint_f32; d.joint_f64 = nullptr; d.joint_f16 = v.joint_f16;
    d.out = t == 0 ? (void*)kd : (void*)vd;
    d.error_word = err;
    const int rc = hqmq_decode(&d, st);
    if (rc != HQMQ_OK) return rc;
  }
  FaParams p;
  p.B = a->batch; p.Hq = a->q_heads; p.Hkv = a->kv_heads; p.Tq = a->q_tokens; p.Tkv = a->kv_tokens;
  p.g = (int)(a->q_heads / a->kv_heads); p.causal = a->causal;
  p.scale_log2 = (float)(a->scale * 1.4426950408889634);
  p.q = a->q; p.k = kd; p.v = vd; p.out = a->out;
  const size_t smem = kQBytes + 5 * (size_t)kKBytes;  // Q, 2 x (K, V), P
  cudaFuncSetAttribute(attention_fa_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int64_t tpt = kFaRows / p.g;
  const dim3 grid((unsigned)ceil_div(a->q_tokens, tpt), (unsigned)(a->batch * a->kv_heads));
  attention_fa_tc_kernel<<<grid, kFaThreads, smem, st>>>(p);
  return check_launch();
}

}  // namespace hqmq
