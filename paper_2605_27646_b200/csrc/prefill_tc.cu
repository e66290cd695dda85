// Prefill attention on the 5th-gen tensor cores (the
// paper's weakest number).  Prefill reads every key many
// times (once per query tile), so the compressed K / V are decoded ONCE into
// an fp16 workspace by the HBM-bound decode kernels, rearranged into the UMMA
// canonical tile layouts (fa_tile_kernel), and flash attention runs over them
// with hand-written tcgen05 MMAs (SWIZZLE_NONE descriptors, one issuing
// thread, tcgen05.commit -> mbarrier, fp32 S and O in TMEM, P written back to
// TMEM as the A operand of the PV MMA).  Two kernels, picked by key count
// (launch_prefill_tc):
//   attention_fa4_kernel  default from 4096 keys: 128-key tiles, two CTAs per
//                         SM, each a sequential S -> softmax -> PV pipeline
//   attention_fa2_kernel  default below: 64-key tiles, two query tiles per CTA,
//                         double-buffered S, TMA producer warps
// Design notes and measurements: DESIGN.md §4 (prefill attention).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

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

// ------------------------------------------------------------------------
// Warp-specialised two-tile version (default below 4096 keys; measured against
// the one-tile 128-key kernel below: 0.090 / 0.71 / 0.84 ms vs 0.099 / 0.66 /
// 0.85 ms on B=1 T=2k / B=1 T=8k / B=4 T=4k).  CTA = 2 query tiles of 128 rows (256
// rows = (256 / g) tokens x g heads of one kv head), 11 warps:
//   warps 0-3 / 4-7  softmax of query tile 0 / 1 (thread = row = TMEM lane)
//   warps 8 / 10     K / V producers: one 1-D bulk copy (TMA) per tile from the
//                    workspace, where the decode left them pre-arranged in the
//                    UMMA canonical layouts (16 KB per 64-key tile)
//   warp 9           MMA issuer (one thread)
// TMEM (512 columns): S0 double buffer [0,128), S1 [128,256), O0 [256,384),
// O1 [384,512).  MMA order S0(0) S1(0) S0(1) S1(1) | PV0(t) S0(t+2) PV1(t)
// S1(t+2) | ...: each group's scores run two tiles ahead of its softmax (one
// mbarrier per S buffer), so the groups drift half a period apart and one
// group's TMEM reads / exponentials overlap the other's, and the tensor cores
// always have the next tile's scores queued.  A 6-stage
// K ring and a 4-stage V ring (full / empty mbarriers; a stage is released by
// tcgen05.commit after the last MMA that reads it; one mbarrier per S / P buffer, as a softmax
// group may finish tile t+1 before the issuer has consumed P(t)).  P is written back into TMEM over its S tile
// and is the A operand of the PV MMA (no shared-memory round trip: the SS
// MMAs are shared-memory-bandwidth bound, 128 B/clk, tools/ubench_umma_tput).
// The running max is only raised when a row's
// tile max exceeds it by more than 8 (log2 domain): exponents stay <= 2^8 in
// fp16 P, O is rescaled in TMEM far less often, and O / l is unchanged.
constexpr int kF2Keys = 64, kF2KStages = 6, kF2VStages = 4, kF2Threads = 352;
constexpr uint32_t kF2TileBytes = kF2Keys * kFaD * 2;  // 16 KB
constexpr uint32_t kF2QOff = 0, kF2KOff = 2 * kQBytes;
constexpr uint32_t kF2VOff = kF2KOff + kF2KStages * kF2TileBytes;
constexpr uint32_t kF2Smem = kF2VOff + kF2VStages * kF2TileBytes;

struct Fa2Params {
  int64_t B, Hq, Hkv, Tq, Tkv, ntk;
  int g, causal;
  float scale_log2;
  const float* q;
  const unsigned char* kt;  // [B*Hkv][ntk] K tiles, K-major canonical
  const unsigned char* vt;  // [B*Hkv][ntk] V tiles, MN-major canonical
  float* out;
};

// mbarrier wait without a suspend-time hint (pure try_wait polling)
__device__ __forceinline__ void fa_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tFA_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@!P1 bra FA_WAIT;\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Softmax inner step over 32 scores of one row (log2 domain): masked entries
// already -inf; exponentials against m_use by ex2.approx (inputs <= 8 or
// -inf), packed fp32 adds, four independent max chains and two sum chains so
// a single warp per SM sub-partition is not latency-bound on them.
__device__ __forceinline__ float fa_ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ void fa_softmax32(const uint32_t (&sr)[32], float m_use, float (&mx)[4],
                                             float2 (&acc)[2], uint32_t* hw) {
  const float2 nm = make_float2(-m_use, -m_use);
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const float s0 = __uint_as_float(sr[2 * e]), s1 = __uint_as_float(sr[2 * e + 1]);
    mx[e & 3] = fmaxf(mx[e & 3], fmaxf(s0, s1));
    const float2 d = __fadd2_rn(make_float2(s0, s1), nm);
    const float e0 = fa_ex2(d.x), e1 = fa_ex2(d.y);
    acc[e & 1] = __fadd2_rn(acc[e & 1], make_float2(e0, e1));
    const __half2 h = __floats2half2_rn(e0, e1);
    hw[e] = *reinterpret_cast<const uint32_t*>(&h);
  }
}

__global__ void __launch_bounds__(kF2Threads, 1) attention_fa2_kernel(Fa2Params p) {
  extern __shared__ __align__(1024) unsigned char fsm[];
  __shared__ __align__(8) uint64_t full_k[kF2KStages], empty_k[kF2KStages];
  __shared__ __align__(8) uint64_t full_v[kF2VStages], empty_v[kF2VStages];
  __shared__ __align__(8) uint64_t bar_s[2][2], bar_p[2][2], bar_o[2], bar_fin;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // grid (B*Hkv, query tiles): concurrently resident CTAs spread over the kv
  // heads (their K / V tiles live in different L2 lines), and the longest
  // causal query tiles start first
  const int64_t bh = blockIdx.x;
  const int64_t b = bh / p.Hkv, hkv = bh % p.Hkv;
  const int g = p.g;
  const int tpt = 2 * kFaRows / g;
  const int64_t tok0 = (int64_t)(gridDim.y - 1 - blockIdx.y) * tpt;
  const int64_t off = p.causal ? (p.Tkv - p.Tq) : 0;
  const int64_t last_tok = std::min(p.Tq, tok0 + tpt) - 1;
  const int64_t kend = p.causal ? std::min(p.Tkv, last_tok + off + 1) : p.Tkv;
  const int ntiles = kend > 0 ? (int)((kend + kF2Keys - 1) / kF2Keys) : 0;

  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "n"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < kF2KStages; ++i) {
      mbar_init(&full_k[i], 1);
      mbar_init(&empty_k[i], 1);
    }
    for (int i = 0; i < kF2VStages; ++i) {
      mbar_init(&full_v[i], 1);
      mbar_init(&empty_v[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bar_s[i][0], 1);
      mbar_init(&bar_s[i][1], 1);
      mbar_init(&bar_p[i][0], kFaRows);
      mbar_init(&bar_p[i][1], kFaRows);
      mbar_init(&bar_o[i], 1);
    }
    mbar_init(&bar_fin, 1);
    fence_mbar_init();
  }
  // softmax threads: this thread's row and its Q row -> fp16 (pre-scaled) A operand
  const int wg = tid >> 7, r = tid & 127;
  const int crow = wg * kFaRows + r;
  const int64_t qtok = tok0 + crow / g;
  const int qhead = crow % g;
  const bool rvalid = tid < 2 * kFaRows && qtok < p.Tq;
  const int64_t vis = p.causal ? std::min(qtok + off + 1, p.Tkv) : p.Tkv;
  if (tid < 2 * kFaRows) {
    unsigned char* qs = fsm + kF2QOff + wg * kQBytes;
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
      *reinterpret_cast<uint4*>(qs + (r >> 3) * kSboQK + kg * 128 + (r & 7) * 16) =
          make_uint4(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1),
                     *reinterpret_cast<const uint32_t*>(&h2), *reinterpret_cast<const uint32_t*>(&h3));
    }
  }
  fence_proxy_async();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_slot;
  const uint32_t sbase = smem_u32(fsm);
  auto k_smem = [&](int t) { return kF2KOff + (uint32_t)(t % kF2KStages) * kF2TileBytes; };
  auto v_smem = [&](int t) { return kF2VOff + (uint32_t)(t % kF2VStages) * kF2TileBytes; };

  if (warp == 8 || warp == 10) {
    // ---- producers (K: warp 8, V: warp 10), one 16 KB bulk copy per tile.
    // Separate rings: a K stage is free once both S MMAs have read it, a V
    // stage only after both PV MMAs, so K runs further ahead.
    if (lane == 0) {
      const bool is_k = warp == 8;
      const int ns = is_k ? kF2KStages : kF2VStages;
      uint64_t* fullb = is_k ? full_k : full_v;
      uint64_t* emptyb = is_k ? empty_k : empty_v;
      const unsigned char* src = (is_k ? p.kt : p.vt) + (size_t)bh * p.ntk * kF2TileBytes;
      for (int t = 0; t < ntiles; ++t) {
        const int st = t % ns;
        if (t >= ns) fa_wait(&emptyb[st], (uint32_t)((t / ns) - 1) & 1u);
        mbar_arrive_expect_tx(&fullb[st], kF2TileBytes);
        bulk_g2s(fsm + (is_k ? k_smem(t) : v_smem(t)), src + (size_t)t * kF2TileBytes, kF2TileBytes,
                 &fullb[st]);
      }
    }
    __syncwarp();
  } else if (warp == 9) {
    // ---- MMA issuer
    if (lane == 0 && ntiles > 0) {
      auto s_mma = [&](int i, int t) {  // S_i(t) = Q_i K(t)^T -> TMEM cols 128 i + 64 (t & 1)
#pragma unroll
        for (int kk = 0; kk < kFaD / 16; ++kk)
          fa_mma(tm + (uint32_t)i * 128 + (uint32_t)(t & 1) * 64, fa_desc(sbase + kF2QOff + i * kQBytes + kk * 256, kSboQK),
                 fa_desc(sbase + k_smem(t) + kk * 256, kSboQK), fa_idesc(kFaRows, kF2Keys, 0),
                 kk > 0);
        fa_commit(&bar_s[i][t & 1]);
        if (i == 1) fa_commit(&empty_k[t % kF2KStages]);
      };
      // O_i += P_i V(t) -> TMEM cols 256 + 128 i; A = P_i(t) from TMEM (fp16
      // pairs written over S_i(t): lane = row, column c = keys 2c, 2c+1)
      auto pv_mma = [&](int i, int t) {
        const uint32_t pa = tm + (uint32_t)i * 128 + (uint32_t)(t & 1) * 64;
#pragma unroll
        for (int kk = 0; kk < kF2Keys / 16; ++kk)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(
                  tm + 256 + (uint32_t)i * 128),
              "r"(pa + kk * 8), "l"(fa_desc(sbase + v_smem(t) + kk * 256, kSboV)),
              "r"(fa_idesc(kFaRows, kFaD, 1)), "r"((t > 0 || kk > 0) ? 1u : 0u));
        fa_commit(&bar_o[i]);
      };
      for (int t = 0; t < 2 && t < ntiles; ++t) {
        fa_wait(&full_k[t], 0);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        s_mma(0, t);
        s_mma(1, t);
      }
      for (int t = 0; t < ntiles; ++t) {
        const uint32_t ph = (uint32_t)t & 1u;
        const bool ahead = t + 2 < ntiles;
        // group i finished with S buffer t & 1 when it arrived with P_i(t)
        fa_wait(&full_v[t % kF2VStages], (uint32_t)(t / kF2VStages) & 1u);
        fa_wait(&bar_p[0][t & 1], (uint32_t)(t >> 1) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        pv_mma(0, t);
        if (ahead) {
          fa_wait(&full_k[(t + 2) % kF2KStages], (uint32_t)((t + 2) / kF2KStages) & 1u);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          s_mma(0, t + 2);
        }
        fa_wait(&bar_p[1][t & 1], (uint32_t)(t >> 1) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        pv_mma(1, t);
        fa_commit(&empty_v[t % kF2VStages]);
        if (ahead) s_mma(1, t + 2);
      }
      // every MMA done (the softmax groups skip PV waits, so bar_o may lag
      // more than one phase behind them)
      fa_commit(&bar_fin);
    }
    __syncwarp();
  } else {
    // ---- softmax (warps 0-7): thread = row r of query tile wg
    const uint32_t tm_row = tm + ((uint32_t)((warp & 3) * 32) << 16);
    const uint32_t o_col = 256 + (uint32_t)wg * 128;
    float m_run = -INFINITY, l_run = 0.f;
    for (int t = 0; t < ntiles; ++t) {
      const uint32_t ph = (uint32_t)t & 1u;
      const int64_t k0 = (int64_t)t * kF2Keys;
      fa_wait(&bar_s[wg][t & 1], (uint32_t)(t >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t s_col = (uint32_t)wg * 128 + ph * 64;
      uint32_t sr[64];
      FA_LD32(tm_row + s_col, sr);
      FA_LD32(tm_row + s_col + 32, (sr + 32));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      if (!rvalid || k0 + kF2Keys > vis) {  // causal / tail / padding-row mask
#pragma unroll
        for (int j = 0; j < 64; ++j)
          if (!rvalid || k0 + j >= vis) sr[j] = __float_as_uint(-INFINITY);
      }
      float mx4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
      for (int j = 0; j < 64; j += 2)
        mx4[(j >> 1) & 3] = fmaxf(mx4[(j >> 1) & 3], fmaxf(__uint_as_float(sr[j]), __uint_as_float(sr[j + 1])));
      const float mx = fmaxf(fmaxf(mx4[0], mx4[1]), fmaxf(mx4[2], mx4[3]));
      const float m_new = (mx > m_run + 8.f) ? mx : m_run;  // also true when m_run = -inf
      const float alpha = (m_new == m_run) ? 1.f : exp2f(m_run - m_new);
      const float m_use = m_new == -INFINITY ? 0.f : m_new;  // all-masked row: exp2(-inf) = 0
      uint32_t hw[32];
      float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
      const float2 nm = make_float2(-m_use, -m_use);
#pragma unroll
      for (int e = 0; e < 32; ++e) {
        const float2 d = __fadd2_rn(make_float2(__uint_as_float(sr[2 * e]), __uint_as_float(sr[2 * e + 1])), nm);
        const float e0 = fa_ex2(d.x), e1 = fa_ex2(d.y);
        acc[e & 1] = __fadd2_rn(acc[e & 1], make_float2(e0, e1));
        const __half2 h = __floats2half2_rn(e0, e1);
        hw[e] = *reinterpret_cast<const uint32_t*>(&h);
      }
      const float psum = (acc[0].x + acc[0].y) + (acc[1].x + acc[1].y);
      l_run = l_run * alpha + psum;
      m_run = m_new;
      // O is only touched when some row's max moved: then PV(t-1) must be done
      // (S(t) completing implies PV(t-2) done, so bar_o is at most one phase behind)
      if (t > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {
        fa_wait(&bar_o[wg], ph ^ 1u);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t orr[32];
            FA_LD32(tm_row + o_col + c * 32, orr);
            asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
            for (int j = 0; j < 32; ++j) orr[j] = __float_as_uint(__uint_as_float(orr[j]) * alpha);
            FA_ST32(tm_row + o_col + c * 32, orr);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
      }
      // P(t) over the first 32 columns of S(t) (already read out)
      FA_ST32(tm_row + s_col, hw);
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&bar_p[wg][t & 1]);
    }
    if (ntiles > 0) {
      fa_wait(&bar_fin, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    float* orow = p.out + ((b * p.Hq + hkv * g + qhead) * p.Tq + (rvalid ? qtok : 0)) * kFaD;
    const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t orr[32];
      if (ntiles > 0) {
        FA_LD32(tm_row + o_col + c * 32, orr);
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
  if (warp == 9)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(512));
}

// ------------------------------------------------------------------------
// 128-key tile geometry shared by the two-CTAs-per-SM kernel below.
constexpr int kF3Keys = 128;
constexpr uint32_t kF3TileBytes = kF3Keys * kFaD * 2;  // 32 KB
constexpr uint32_t kSbo128 = (kF3Keys / 8) * 128;  // MN-major V: 16 key-groups per 8-dim group

#define FA_ST16(addr, r)                                                                        \
  asm volatile(                                                                                 \
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12," \
      "%13,%14,%15,%16};" ::"r"(addr),                                                        \
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),  \
      "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]),         \
      "r"(r[15]))

// ------------------------------------------------------------------------
// Two-CTAs-per-SM version (default from 4096 keys).  Each CTA is one strictly
// sequential pipeline over 128-key tiles -- S(t) -> softmax(t) -> PV(t) ->
// S(t+1) -- and the two co-resident CTAs interleave on the SM's tensor cores,
// MUFU and TMEM ports, so one CTA's softmax hides the other's MMAs (and each
// CTA's prologue / epilogue hides behind the other's steady state).
// CTA = 128 query rows, 10 warps: softmax 0-7 (warps w and w+4 share TMEM
// lanes 32 (w % 4) and split each row's 128 keys), producer 8 (K then V, one
// stage each: K(t+1) streams in during softmax(t), V(t+1) during S(t+1)),
// MMA issuer 9.  TMEM 256 columns: S [0,128) with P(t) over
// its first 64, O [128,256).  Because S(t) is issued after PV(t-1), S(t)
// complete implies O is idle: the softmax rescales O without any wait.
constexpr int kF4Threads = 320;
constexpr uint32_t kF4KOff = kQBytes, kF4VOff = kQBytes + kF3TileBytes;
constexpr uint32_t kF4Smem = kQBytes + 2 * kF3TileBytes;  // 96 KB: two CTAs per SM

__global__ void __launch_bounds__(kF4Threads, 2) attention_fa4_kernel(Fa2Params p) {
  extern __shared__ __align__(1024) unsigned char fsm[];
  __shared__ __align__(8) uint64_t full_k, empty_k, full_v, empty_v, bar_s, bar_p, bar_fin;
  __shared__ uint32_t tmem_slot;
  __shared__ float xch[2][kFaRows];  // per-half tile max / final l exchange
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t bh = blockIdx.x;
  const int64_t b = bh / p.Hkv, hkv = bh % p.Hkv;
  const int g = p.g;
  const int tpt = kFaRows / g;
  const int64_t tok0 = (int64_t)(gridDim.y - 1 - blockIdx.y) * tpt;
  const int64_t off = p.causal ? (p.Tkv - p.Tq) : 0;
  const int64_t last_tok = std::min(p.Tq, tok0 + tpt) - 1;
  const int64_t kend = p.causal ? std::min(p.Tkv, last_tok + off + 1) : p.Tkv;
  const int ntiles = kend > 0 ? (int)((kend + kF3Keys - 1) / kF3Keys) : 0;

  if (warp == 9) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&tmem_slot)),
                 "n"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(&full_k, 1);
    mbar_init(&empty_k, 1);
    mbar_init(&full_v, 1);
    mbar_init(&empty_v, 1);
    mbar_init(&bar_s, 1);
    mbar_init(&bar_p, 2 * kFaRows);
    mbar_init(&bar_fin, 1);
    fence_mbar_init();
  }
  const int r = tid & 127, half = (tid >> 7) & 1;
  const int64_t qtok = tok0 + r / g;
  const int qhead = r % g;
  const bool rvalid = tid < 2 * kFaRows && qtok < p.Tq;
  const int64_t vis = p.causal ? std::min(qtok + off + 1, p.Tkv) : p.Tkv;
  if (tid < kFaRows) {
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
      *reinterpret_cast<uint4*>(fsm + (r >> 3) * kSboQK + kg * 128 + (r & 7) * 16) =
          make_uint4(*reinterpret_cast<const uint32_t*>(&h0), *reinterpret_cast<const uint32_t*>(&h1),
                     *reinterpret_cast<const uint32_t*>(&h2), *reinterpret_cast<const uint32_t*>(&h3));
    }
  }
  fence_proxy_async();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tmem_slot;
  const uint32_t sbase = smem_u32(fsm);

  if (warp == 8) {
    // ---- producer: K(t) when S(t-1) has read the K stage, V(t) when PV(t-1)
    // has read the V stage
    if (lane == 0) {
      const unsigned char* kb = p.kt + (size_t)bh * p.ntk * kF3TileBytes;
      const unsigned char* vb = p.vt + (size_t)bh * p.ntk * kF3TileBytes;
      for (int t = 0; t < ntiles; ++t) {
        if (t > 0) fa_wait(&empty_k, (uint32_t)(t - 1) & 1u);
        mbar_arrive_expect_tx(&full_k, kF3TileBytes);
        bulk_g2s(fsm + kF4KOff, kb + (size_t)t * kF3TileBytes, kF3TileBytes, &full_k);
        if (t > 0) fa_wait(&empty_v, (uint32_t)(t - 1) & 1u);
        mbar_arrive_expect_tx(&full_v, kF3TileBytes);
        bulk_g2s(fsm + kF4VOff, vb + (size_t)t * kF3TileBytes, kF3TileBytes, &full_v);
      }
    }
    __syncwarp();
  } else if (warp == 9) {
    // ---- MMA issuer
    if (lane == 0 && ntiles > 0) {
      for (int t = 0; t < ntiles; ++t) {
        const uint32_t ph = (uint32_t)t & 1u;
        fa_wait(&full_k, ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int kk = 0; kk < kFaD / 16; ++kk)
          fa_mma(tm, fa_desc(sbase + kk * 256, kSboQK), fa_desc(sbase + kF4KOff + kk * 256, kSboQK),
                 fa_idesc(kFaRows, kF3Keys, 0), kk > 0);
        fa_commit(&bar_s);
        fa_commit(&empty_k);
        fa_wait(&bar_p, ph);
        fa_wait(&full_v, ph);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll
        for (int kk = 0; kk < kF3Keys / 16; ++kk)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tm + 128),
              "r"(tm + kk * 8), "l"(fa_desc(sbase + kF4VOff + kk * 256, kSbo128)),
              "r"(fa_idesc(kFaRows, kFaD, 1)), "r"((t > 0 || kk > 0) ? 1u : 0u));
        fa_commit(&empty_v);
      }
      fa_commit(&bar_fin);
    }
    __syncwarp();
  } else {
    // ---- softmax (warps 0-7): thread = (row r, key half); warps w and w+4
    // share TMEM lanes 32 (w % 4) and exchange tile maxima / l in shared memory
    const uint32_t tm_row = tm + ((uint32_t)((warp & 3) * 32) << 16);
    const uint32_t o_col = 128 + (uint32_t)half * 64;
    const int pair_bar = 1 + (warp & 3);
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory"); };
    float m_run = -INFINITY, l_run = 0.f;
    for (int t = 0; t < ntiles; ++t) {
      const int64_t k0 = (int64_t)t * kF3Keys + half * 64;
      fa_wait(&bar_s, (uint32_t)t & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const bool mask = !rvalid || k0 + 64 > vis;
      uint32_t hw[32];
      auto pass = [&](float m_use, float& tile_max) {
        float mx[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
        float2 acc[2] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t sr[32];
          FA_LD32(tm_row + half * 64 + c * 32, sr);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (mask) {
#pragma unroll
            for (int j = 0; j < 32; ++j)
              if (!rvalid || k0 + c * 32 + j >= vis) sr[j] = __float_as_uint(-INFINITY);
          }
          fa_softmax32(sr, m_use, mx, acc, hw + c * 16);
        }
        tile_max = fmaxf(fmaxf(mx[0], mx[1]), fmaxf(mx[2], mx[3]));
        return (acc[0].x + acc[0].y) + (acc[1].x + acc[1].y);
      };
      float tmax = -INFINITY;
      float psum = pass(m_run == -INFINITY ? 0.f : m_run, tmax);
      xch[half][r] = tmax;
      pair_sync();
      tmax = fmaxf(tmax, xch[half ^ 1][r]);
      const bool jump = tmax > m_run + 8.f;  // same in both halves of the row
      const float m_new = jump ? tmax : m_run;
      if (__any_sync(0xffffffffu, jump)) {  // warp-uniform (.sync.aligned loads)
        float dummy = -INFINITY;
        psum = pass(m_new == -INFINITY ? 0.f : m_new, dummy);
      }
      pair_sync();  // both halves done reading S(t) before P overwrites it
#pragma unroll
      for (int c = 0; c < 2; ++c) FA_ST16(tm_row + half * 32 + c * 16, (hw + c * 16));
      const float alpha = (m_new == m_run) ? 1.f : exp2f(m_run - m_new);
      l_run = l_run * alpha + psum;
      m_run = m_new;
      if (t > 0 && __any_sync(0xffffffffu, alpha != 1.f)) {  // O idle: S(t) done => PV(t-1) done
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t orr[32];
          FA_LD32(tm_row + o_col + c * 32, orr);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 32; ++j) orr[j] = __float_as_uint(__uint_as_float(orr[j]) * alpha);
          FA_ST32(tm_row + o_col + c * 32, orr);
        }
      }
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&bar_p);
    }
    pair_sync();
    xch[half][r] = l_run;
    pair_sync();
    l_run += xch[half ^ 1][r];
    if (ntiles > 0) {
      fa_wait(&bar_fin, 0);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    }
    float* orow = p.out + ((b * p.Hq + hkv * g + qhead) * p.Tq + (rvalid ? qtok : 0)) * kFaD + half * 64;
    const float inv = l_run > 0.f ? 1.f / l_run : 0.f;
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      uint32_t orr[32];
      if (ntiles > 0) {
        FA_LD32(tm_row + o_col + c * 32, orr);
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
  if (warp == 9)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "n"(256));
}

// Linear decoded fp16 (B*Hkv, T, 128) -> kt-key UMMA tiles (16-byte units):
//   K-major (K):  unit(key, dg) at (key/8)*128 + dg*8 + key%8
//   MN-major (V): unit(key, dg) at dg*kt + (key/8)*8 + key%8
// keys past T are zero-filled (masked P = 0 must not meet a NaN in V).
__global__ void fa_tile_kernel(const uint4* __restrict__ lin, uint4* __restrict__ tiles, int64_t BH,
                               int64_t T, int64_t ntk, int mn_major, int kt) {
  const int64_t per_bh = ntk * kt * 16;
  const int64_t n = BH * per_bh;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int dg = (int)(i & 15);
    const int64_t bh = i / per_bh, tok = (i - bh * per_bh) >> 4;
    const uint4 v = tok < T ? __ldg(lin + (bh * T + tok) * 16 + dg) : make_uint4(0u, 0u, 0u, 0u);
    const int key = (int)(tok % kt);
    const int64_t tile = tok / kt;
    const int o = mn_major ? dg * kt + (key >> 3) * 8 + (key & 7) : (key >> 3) * 128 + dg * 8 + (key & 7);
    tiles[(bh * ntk + tile) * (kt * 16) + o] = v;
  }
}

// Zero the units of keys >= T in every row's last tile (K and V tiles), so the
// masked P = 0 never meets a NaN from uninitialised workspace.
__global__ void fa_pad_kernel(uint4* __restrict__ kt, uint4* __restrict__ vt, int64_t BH, int64_t T,
                              int64_t ntk, int keys) {
  const int first = (int)(T % keys), npad = keys - first;
  const int64_t n = BH * npad * 16;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int dg = (int)(i & 15);
    const int64_t bh = (i >> 4) / npad;
    const int key = first + (int)((i >> 4) - bh * npad);
    const int64_t base = (bh * ntk + ntk - 1) * (int64_t)keys * 16;
    kt[base + (key >> 3) * 128 + dg * 8 + (key & 7)] = make_uint4(0u, 0u, 0u, 0u);
    vt[base + dg * keys + (key >> 3) * 8 + (key & 7)] = make_uint4(0u, 0u, 0u, 0u);
  }
}

// decode.cu: fast decode straight into UMMA tiles (HQMQ_ERR_UNSUPPORTED when
// it does not apply)
int decode_fp16_tiles(const hqmq_decode_args* a, int tile_log2, int mn, int64_t ntk, void* tiles,
                      cudaStream_t st);

// Decode-once + tcgen05 flash attention for prefill shapes.  Workspace: the
// two decoded fp16 tensors (kv layout) + an error word.
size_t prefill_tc_workspace(const hqmq_attention_args* a) {
  const size_t bh = (size_t)a->batch * a->kv_heads;
  const size_t lin = 2 * bh * a->kv_tokens * kFaD * 2;
  const size_t tiles = 2 * bh * std::max((size_t)ceil_div(a->kv_tokens, kF2Keys) * kF2TileBytes,
                                         (size_t)ceil_div(a->kv_tokens, kF3Keys) * kF3TileBytes);
  return lin + tiles + 256;
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
  hqmq_decode_args dargs[2];
  for (int t = 0; t < 2; ++t) {
    const hqmq_packed_view& v = t == 0 ? a->k : a->v;
    hqmq_decode_args& d = dargs[t];
    d = hqmq_decode_args{};
    d.batch = a->batch; d.heads = a->kv_heads; d.tokens = a->kv_tokens; d.head_dim = a->head_dim;
    d.codebook_size = a->codebook_size; d.radius_bits = a->radius_bits; d.index_bits = a->index_bits;
    d.out_dtype = HQMQ_F16;
    d.token_start = 0; d.token_stop = a->kv_tokens;
    d.scales = v.scales; d.index_words = v.index_words; d.radius_words = v.radius_words;
    d.flag_words = v.flag_words; d.payloads = v.payloads; d.token_offsets = v.token_offsets;
    d.joint_f32 = v.joint_f32; d.joint_f64 = nullptr; d.joint_f16 = v.joint_f16;
    d.out = t == 0 ? (void*)kd : (void*)vd;
    d.error_word = err;
  }
  auto decode_rowmajor = [&]() {
    for (int t = 0; t < 2; ++t) {
      const int rc = hqmq_decode(&dargs[t], st);
      if (rc != HQMQ_OK) return rc;
    }
    return (int)HQMQ_OK;
  };
  // the two-CTAs-per-SM 128-key kernel for long key ranges (0.62 ms at 8k vs
  // 0.71 for the two-tile 64-key kernel), the 64-key kernel for short ones
  // (0.090 vs 0.093 ms at 2k)
  const bool v4 = a->kv_tokens >= 4096;
  const int keys = v4 ? kF3Keys : kF2Keys;
  const uint32_t tile_bytes = v4 ? kF3TileBytes : kF2TileBytes;
  const int64_t bh = a->batch * a->kv_heads;
  const int64_t ntk = ceil_div(a->kv_tokens, keys);
  unsigned char* kt = ws + 2 * nelem * 2;
  unsigned char* vt = kt + (size_t)bh * ntk * tile_bytes;
  // the fast decode writes its 16-byte units straight into the tiles; other
  // streams (Med3x) decode row-major and are re-laid out
  const int log2k = v4 ? 7 : 6;
  int rc = decode_fp16_tiles(&dargs[0], log2k, 0, ntk, kt, st);
  if (rc == HQMQ_OK) rc = decode_fp16_tiles(&dargs[1], log2k, 1, ntk, vt, st);
  if (rc == HQMQ_OK) {
    if (a->kv_tokens % keys) {  // keys past T in each row's last tile: zeros
      const int64_t units = bh * (keys - a->kv_tokens % keys) * 16;
      fa_pad_kernel<<<(unsigned)std::min<int64_t>(ceil_div(units, 256), 148 * 16), 256, 0, st>>>(
          reinterpret_cast<uint4*>(kt), reinterpret_cast<uint4*>(vt), bh, a->kv_tokens, ntk, keys);
    }
  } else if (rc == HQMQ_ERR_UNSUPPORTED) {
    rc = decode_rowmajor();
    if (rc != HQMQ_OK) return rc;
    const int64_t units = bh * ntk * keys * 16;
    const unsigned grid_t = (unsigned)std::min<int64_t>(ceil_div(units, 256), 148 * 16);
    fa_tile_kernel<<<grid_t, 256, 0, st>>>(reinterpret_cast<const uint4*>(kd), reinterpret_cast<uint4*>(kt),
                                           bh, a->kv_tokens, ntk, 0, keys);
    fa_tile_kernel<<<grid_t, 256, 0, st>>>(reinterpret_cast<const uint4*>(vd), reinterpret_cast<uint4*>(vt),
                                           bh, a->kv_tokens, ntk, 1, keys);
  } else {
    return rc;
  }
  rc = check_launch();
  if (rc != HQMQ_OK) return rc;
  Fa2Params q2;
  q2.B = a->batch; q2.Hq = a->q_heads; q2.Hkv = a->kv_heads; q2.Tq = a->q_tokens;
  q2.Tkv = a->kv_tokens; q2.ntk = ntk;
  q2.g = (int)(a->q_heads / a->kv_heads); q2.causal = a->causal;
  q2.scale_log2 = (float)(a->scale * 1.4426950408889634);
  q2.q = a->q; q2.kt = kt; q2.vt = vt; q2.out = a->out;
  if (v4) {
    cudaFuncSetAttribute(attention_fa4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kF4Smem);
    const dim3 grid((unsigned)bh, (unsigned)ceil_div(a->q_tokens, kFaRows / q2.g));
    attention_fa4_kernel<<<grid, kF4Threads, kF4Smem, st>>>(q2);
    return check_launch();
  }
  cudaFuncSetAttribute(attention_fa2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kF2Smem);
  const int64_t tpt = 2 * kFaRows / q2.g;
  const dim3 grid((unsigned)bh, (unsigned)ceil_div(a->q_tokens, tpt));
  attention_fa2_kernel<<<grid, kF2Threads, kF2Smem, st>>>(q2);
  return check_launch();
}

}  // namespace hqmq
