// Pure compute rate of the 7x7 stencil's strip block body:
// no TMA, no barriers, no stores -- each warp re-reads a static shared-memory
// window and sums its outputs.  Scalar FFMA (the kernel's form, weights in
// uniform registers) against packed FFMA2 column pairs (fma.rn.f32x2 with the
// tap broadcast from a uniform register, odd-offset pairs built by PRMT),
// H = 4 / 8 output rows per block, 2-4 CTAs of 128 threads per SM.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o body_rate stencil_body_rate.cu
// Measured (one B200, round 2): scalar H=4 65.0-66.5, scalar H=8 67.6-68.6,
// FFMA2 H=4 55.1-58.6, FFMA2 H=8 62.5-63.9 TFLOP/s (FFMA peak 72.5).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
constexpr int R = 3, F = 7, SW = 136, D = 1;
__device__ __forceinline__ uint64_t ffma2_bcast(uint64_t x, float w, uint64_t acc) {
  uint64_t ww;
  asm("mov.b64 %0, {%1, %1};" : "=l"(ww) : "f"(w));
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(x), "l"(ww));
  return acc;
}
__device__ __forceinline__ uint64_t pair_hi_lo(uint64_t a, uint64_t b) {
  uint64_t r;
  asm volatile("{.reg .b32 a0, a1, b0, b1, r0, r1;\n\tmov.b64 {a0, a1}, %1;\n\tmov.b64 {b0, b1}, %2;\n\tprmt.b32 r0, a1, 0, 0x3210;\n\tprmt.b32 r1, b0, 0, 0x3210;\n\tmov.b64 %0, {r0, r1};}" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
template <int H, bool F2>
__global__ void __launch_bounds__(128) k(float *out, const float *wg, int iters, int rows) {
  extern __shared__ __align__(16) float win[];
  __shared__ float w[49];
  for (int e = threadIdx.x; e < 49; e += blockDim.x) w[e] = wg[e];
  for (int e = threadIdx.x; e < 4 * SW * 24; e += blockDim.x) win[e] = (e % 97) * 0.01f;
  __syncthreads();
  float wr[49];
#pragma unroll
  for (int e = 0; e < 49; ++e) wr[e] = w[e];
  const int u = threadIdx.x;
  const float *sbase = win + (u >> 5) * (SW * 24) + (u & 31) * 4;
  float sink = 0.f;
#pragma unroll 1
  for (int it = 0; it < iters; ++it) {
#pragma unroll 1
    for (int r0 = 0; r0 < rows; r0 += H) {
      const int rb = (r0 + it) & 7;
      if constexpr (F2) {
        uint64_t acc[H][2];
#pragma unroll
        for (int h = 0; h < H; ++h) acc[h][0] = acc[h][1] = 0ull;
#pragma unroll
        for (int p = 0; p < H + F - 1; ++p) {
          uint64_t ev[6];
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const ulonglong2 t2 = *reinterpret_cast<const ulonglong2 *>(sbase + (rb + p) * SW + 4 * q);
            ev[2 * q] = t2.x; ev[2 * q + 1] = t2.y;
          }
          uint64_t od[5];
#pragma unroll
          for (int m = 0; m < 5; ++m) od[m] = pair_hi_lo(ev[m], ev[m + 1]);
#pragma unroll
          for (int q = 0; q < F; ++q)
#pragma unroll
            for (int h = 0; h < H; ++h) {
              const int pp = p - h;
              if (pp >= 0 && pp < F) {
#pragma unroll
                for (int m = 0; m < 2; ++m) {
                  const int kk = 2 * m + q + D;
                  acc[h][m] = ffma2_bcast(kk % 2 == 0 ? ev[kk / 2] : od[kk / 2], wr[pp * F + q], acc[h][m]);
                }
              }
            }
        }
#pragma unroll
        for (int h = 0; h < H; ++h) {
          float a0, a1, b0, b1;
          asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(acc[h][0]));
          asm("mov.b64 {%0, %1}, %2;" : "=f"(b0), "=f"(b1) : "l"(acc[h][1]));
          sink += a0 + a1 + b0 + b1;
        }
      } else {
        float acc[H][4];
#pragma unroll
        for (int h = 0; h < H; ++h)
#pragma unroll
          for (int t = 0; t < 4; ++t) acc[h][t] = 0.f;
#pragma unroll
        for (int p = 0; p < H + F - 1; ++p) {
          float v[12];
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const float4 t4 = *reinterpret_cast<const float4 *>(sbase + (rb + p) * SW + 4 * q);
            v[4 * q] = t4.x; v[4 * q + 1] = t4.y; v[4 * q + 2] = t4.z; v[4 * q + 3] = t4.w;
          }
#pragma unroll
          for (int q = 0; q < F; ++q)
#pragma unroll
            for (int h = 0; h < H; ++h) {
              const int pp = p - h;
              if (pp >= 0 && pp < F) {
#pragma unroll
                for (int t = 0; t < 4; ++t) acc[h][t] = __fmaf_rn(wr[pp * F + q], v[1 + t + q], acc[h][t]);
              }
            }
        }
#pragma unroll
        for (int h = 0; h < H; ++h) sink += acc[h][0] + acc[h][1] + acc[h][2] + acc[h][3];
      }
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = sink;
}
template <int H, bool F2>
void run(const char *name, float *out, float *w, int bps) {
  auto kern = k<H, F2>;
  const int smem = 4 * SW * 24 * 4;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int rows = 8, iters = 4000;
  kern<<<148 * bps, 128, smem>>>(out, w, 10, rows);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  kern<<<148 * bps, 128, smem>>>(out, w, iters, rows);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double fma = 148.0 * bps * 128 * (double)iters * rows * 4 * 49;
  printf("%-14s blocks/SM %d: %.2f TFLOP/s (%s)\n", name, bps, 2 * fma / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
}
int main() {
  float *out, *w;
  cudaMalloc(&out, 148 * 16 * 128 * 4); cudaMalloc(&w, 49 * 4);
  float hw[49]; for (int i = 0; i < 49; ++i) hw[i] = 0.01f * (i + 1);
  cudaMemcpy(w, hw, sizeof hw, cudaMemcpyHostToDevice);
  for (int bps : {2, 3, 4}) {
    run<4, false>("scalar H=4", out, w, bps);
    run<4, true>("ffma2 H=4", out, w, bps);
    run<8, true>("ffma2 H=8", out, w, bps);
    run<8, false>("scalar H=8", out, w, bps);
  }
  return 0;
}
