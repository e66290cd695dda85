// Microbenchmark of the encode S-loop formulations (FP32 pipe), isolated from
// the prologue/pack.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 \
//   -o ubench tools/ubench_encode_loop.cu && ./ubench
// Prints (chunk x secondary) pairs per second and the fraction of the FP32
// roofline (20 lane-ops per pair at 148 SMs x 128 lanes x clock).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <vector>

#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e = (x);                                                          \
    if (e != cudaSuccess) {                                                       \
      printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__);                 \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

__device__ __forceinline__ float max3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// Variant 0: FFMA2 on (w,x)/(y,z) pairs, R chunks per lane, FSETP+SEL argmax.
// Variant 1: as 0 with explicit 3-input max for the 5-way max.
// Variant 2: as 1 with the argmax folded into the score's low mantissa bits
//            (keyed max: one LOP3 instead of FSETP+SEL).
// Variant 3: scalar FFMA (no packed math).
template <int R, int V>
__global__ void __launch_bounds__(256) loop_kernel(const float4* __restrict__ dirs,
                                                   const float4* __restrict__ rot, int S,
                                                   int reps, float* out) {
  extern __shared__ float4 tab[];
  for (int i = threadIdx.x; i < S * 4; i += blockDim.x) tab[i] = rot[i];
  __syncthreads();
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  float u[R][4];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const float4 d = dirs[(gid * R + j) & 4095];
    u[j][0] = d.x; u[j][1] = d.y; u[j][2] = d.z; u[j][3] = d.w;
  }
  float acc = 0.f;
  for (int rep = 0; rep < reps; ++rep) {
    float best[R], second[R];
    int bs[R];
#pragma unroll
    for (int j = 0; j < R; ++j) { best[j] = -1.f; second[j] = -1.f; bs[j] = 0; }
#pragma unroll 2
    for (int s = 0; s < S; ++s) {
      const float4 t0 = tab[4 * s], t1 = tab[4 * s + 1], t2 = tab[4 * s + 2], t3 = tab[4 * s + 3];
#pragma unroll
      for (int j = 0; j < R; ++j) {
        float w, x, y, z;
        if (V == 3) {
          w = u[j][3] * t1.z; w = fmaf(u[j][2], t1.x, w); w = fmaf(u[j][1], t0.z, w); w = fmaf(u[j][0], t0.x, w);
          x = u[j][3] * t1.w; x = fmaf(u[j][2], t1.y, x); x = fmaf(u[j][1], t0.w, x); x = fmaf(u[j][0], t0.y, x);
          y = u[j][3] * t3.z; y = fmaf(u[j][2], t3.x, y); y = fmaf(u[j][1], t2.z, y); y = fmaf(u[j][0], t2.x, y);
          z = u[j][3] * t3.w; z = fmaf(u[j][2], t3.y, z); z = fmaf(u[j][1], t2.w, z); z = fmaf(u[j][0], t2.y, z);
        } else {
          float2 wx = __fmul2_rn(make_float2(u[j][3], u[j][3]), make_float2(t1.z, t1.w));
          wx = __ffma2_rn(make_float2(u[j][2], u[j][2]), make_float2(t1.x, t1.y), wx);
          wx = __ffma2_rn(make_float2(u[j][1], u[j][1]), make_float2(t0.z, t0.w), wx);
          wx = __ffma2_rn(make_float2(u[j][0], u[j][0]), make_float2(t0.x, t0.y), wx);
          float2 yz = __fmul2_rn(make_float2(u[j][3], u[j][3]), make_float2(t3.z, t3.w));
          yz = __ffma2_rn(make_float2(u[j][2], u[j][2]), make_float2(t3.x, t3.y), yz);
          yz = __ffma2_rn(make_float2(u[j][1], u[j][1]), make_float2(t2.z, t2.w), yz);
          yz = __ffma2_rn(make_float2(u[j][0], u[j][0]), make_float2(t2.x, t2.y), yz);
          w = wx.x; x = wx.y; y = yz.x; z = yz.y;
        }
        const float aw = fabsf(w), ax = fabsf(x), ay = fabsf(y), az = fabsf(z);
        float half;
        if (V == 6) {
          const float2 p2 = __fadd2_rn(make_float2(aw, ax), make_float2(ay, az));
          half = (p2.x + p2.y) * 0.5f;
        } else {
          half = ((aw + ax) + (ay + az)) * 0.5f;
        }
        float sc;
        if (V == 0 || V == 3) sc = fmaxf(fmaxf(fmaxf(aw, ax), fmaxf(ay, az)), half);
        else sc = max3(max3(aw, ax, ay), az, half);
        if (V == 5) {  // best only (lower bound on the tracking cost)
          const bool gt = sc > best[j];
          best[j] = fmaxf(best[j], sc);
          bs[j] = gt ? s : bs[j];
        } else if (V == 7) {  // keyed best, plain second
          const float key = __int_as_float((__float_as_int(sc) & ~63) | (s & 63));
          second[j] = fmaxf(second[j], fminf(sc, best[j]));
          best[j] = fmaxf(best[j], key);
        } else if (V == 2) {
          const float key = __int_as_float((__float_as_int(sc) & ~63) | (63 - (s & 63)));
          second[j] = fmaxf(second[j], fminf(key, best[j]));
          best[j] = fmaxf(best[j], key);
        } else {
          const bool gt = sc > best[j];
          second[j] = fmaxf(second[j], fminf(sc, best[j]));
          best[j] = fmaxf(best[j], sc);
          bs[j] = gt ? s : bs[j];
        }
      }
    }
#pragma unroll
    for (int j = 0; j < R; ++j) acc += best[j] - second[j] + (float)bs[j];
  }
  if (acc == 1234.5f) out[gid] = acc;
}


// Variant 8/9: FFMA2 over CHUNK pairs (lanes of the float2 = two chunks), table
// values broadcast: the |v| sums and the x0.5 also run as packed FADD2/FMUL2,
// cutting FMA-pipe issue slots per (chunk, secondary) from 12 to 10.
// 9 = 8 + keyed best (score low bits carry s).
template <int R, int V>
__global__ void __launch_bounds__(256) pair_kernel(const float4* __restrict__ dirs,
                                                   const float4* __restrict__ rot, int S,
                                                   int reps, float* out) {
  extern __shared__ float4 tab[];
  for (int i = threadIdx.x; i < S * 4; i += blockDim.x) tab[i] = rot[i];
  __syncthreads();
  const int gid = blockIdx.x * blockDim.x + threadIdx.x;
  constexpr int P = R / 2;
  float2 U[P][4];
#pragma unroll
  for (int j = 0; j < P; ++j) {
    const float4 d0 = dirs[(gid * R + 2 * j) & 4095], d1 = dirs[(gid * R + 2 * j + 1) & 4095];
    U[j][0] = make_float2(d0.x, d1.x); U[j][1] = make_float2(d0.y, d1.y);
    U[j][2] = make_float2(d0.z, d1.z); U[j][3] = make_float2(d0.w, d1.w);
  }
  float acc = 0.f;
  for (int rep = 0; rep < reps; ++rep) {
    float best[R], second[R];
    int bs[R];
#pragma unroll
    for (int j = 0; j < R; ++j) { best[j] = -1.f; second[j] = -1.f; bs[j] = 0; }
#pragma unroll 2
    for (int s = 0; s < S; ++s) {
      const float4 t0 = tab[4 * s], t1 = tab[4 * s + 1], t2 = tab[4 * s + 2], t3 = tab[4 * s + 3];
#pragma unroll
      for (int j = 0; j < P; ++j) {
        float2 W = __fmul2_rn(U[j][3], make_float2(t1.z, t1.z));
        W = __ffma2_rn(U[j][2], make_float2(t1.x, t1.x), W);
        W = __ffma2_rn(U[j][1], make_float2(t0.z, t0.z), W);
        W = __ffma2_rn(U[j][0], make_float2(t0.x, t0.x), W);
        float2 X = __fmul2_rn(U[j][3], make_float2(t1.w, t1.w));
        X = __ffma2_rn(U[j][2], make_float2(t1.y, t1.y), X);
        X = __ffma2_rn(U[j][1], make_float2(t0.w, t0.w), X);
        X = __ffma2_rn(U[j][0], make_float2(t0.y, t0.y), X);
        float2 Y = __fmul2_rn(U[j][3], make_float2(t3.z, t3.z));
        Y = __ffma2_rn(U[j][2], make_float2(t3.x, t3.x), Y);
        Y = __ffma2_rn(U[j][1], make_float2(t2.z, t2.z), Y);
        Y = __ffma2_rn(U[j][0], make_float2(t2.x, t2.x), Y);
        float2 Z = __fmul2_rn(U[j][3], make_float2(t3.w, t3.w));
        Z = __ffma2_rn(U[j][2], make_float2(t3.y, t3.y), Z);
        Z = __ffma2_rn(U[j][1], make_float2(t2.w, t2.w), Z);
        Z = __ffma2_rn(U[j][0], make_float2(t2.y, t2.y), Z);
        const float2 aW = make_float2(fabsf(W.x), fabsf(W.y)), aX = make_float2(fabsf(X.x), fabsf(X.y));
        const float2 aY = make_float2(fabsf(Y.x), fabsf(Y.y)), aZ = make_float2(fabsf(Z.x), fabsf(Z.y));
        const float2 H = __fmul2_rn(__fadd2_rn(__fadd2_rn(aW, aX), __fadd2_rn(aY, aZ)),
                                    make_float2(0.5f, 0.5f));
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int jj = 2 * j + e;
          const float sc = e ? max3(max3(aW.y, aX.y, aY.y), aZ.y, H.y)
                             : max3(max3(aW.x, aX.x, aY.x), aZ.x, H.x);
          if (V == 9) {
            const float key = __int_as_float((__float_as_int(sc) & ~63) | (s & 63));
            second[jj] = fmaxf(second[jj], fminf(sc, best[jj]));
            best[jj] = fmaxf(best[jj], key);
          } else {
            const bool gt = sc > best[jj];
            second[jj] = fmaxf(second[jj], fminf(sc, best[jj]));
            best[jj] = fmaxf(best[jj], sc);
            bs[jj] = gt ? s : bs[jj];
          }
        }
      }
    }
#pragma unroll
    for (int j = 0; j < R; ++j) acc += best[j] - second[j] + (float)bs[j];
  }
  if (acc == 1234.5f) out[gid] = acc;
}

template <int R, int V>
int run(const char* name, float4* dirs, float4* rot, float* out, int S, int blocks_per_sm);

template <int R, int V>
int run(const char* name, float4* dirs, float4* rot, float* out, int S, int blocks_per_sm) {
  const int smem = S * 64;
  auto kern = V >= 8 ? pair_kernel<R, V> : loop_kernel<R, V>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 256, smem);
  const int blocks = 148 * (blocks_per_sm ? blocks_per_sm : occ);
  const int reps = 40;
  kern<<<blocks, 256, smem>>>(dirs, rot, S, 2, out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  kern<<<blocks, 256, smem>>>(dirs, rot, S, reps, out);
  cudaEventRecord(b);
  CK(cudaEventSynchronize(b));
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double pairs = (double)blocks * 256 * R * S * reps;
  const double lane_ops = pairs * 20;
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double peak = 148.0 * 128 * clk_khz * 1e3;
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  printf("%-28s R=%d occ=%d regs=%3d  %8.3f ms  %7.2f Gpair/s  %6.2f T lane-op/s  frac(max clk)=%.3f\n",
         name, R, occ, fa.numRegs, ms, pairs / ms / 1e6, lane_ops / ms / 1e9, lane_ops / (ms * 1e-3) / peak);
  return 0;
}

int main() {
  const int S = 64;
  std::vector<float> h(4096 * 4), hr(S * 16);
  uint32_t st = 12345;
  auto rnd = [&]() { st = st * 1664525u + 1013904223u; return (st >> 8) * (1.0f / 16777216.0f) - 0.5f; };
  for (auto& v : h) v = rnd();
  for (auto& v : hr) v = rnd();
  float4 *dirs, *rot;
  float* out;
  CK(cudaMalloc(&dirs, h.size() * 4));
  CK(cudaMalloc(&rot, hr.size() * 4));
  CK(cudaMalloc(&out, 148 * 32 * 256 * 4));
  cudaMemcpy(dirs, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(rot, hr.data(), hr.size() * 4, cudaMemcpyHostToDevice);
  run<4, 1>("ffma2 max3", dirs, rot, out, S, 0);
  run<4, 8>("chunk-pair ffma2", dirs, rot, out, S, 0);
  run<4, 9>("chunk-pair ffma2 keyed", dirs, rot, out, S, 0);
  run<8, 8>("chunk-pair ffma2", dirs, rot, out, S, 0);
  run<8, 9>("chunk-pair ffma2 keyed", dirs, rot, out, S, 0);
  run<6, 8>("chunk-pair ffma2", dirs, rot, out, S, 0);
  run<2, 8>("chunk-pair ffma2", dirs, rot, out, S, 0);
  return 0;
}
