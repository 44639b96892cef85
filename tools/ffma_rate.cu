// Microbenchmark: FFMA issue rate by operand form (3 registers, kernel-param
// constant operand, immediate).  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>

template <int FORM>
__global__ void __launch_bounds__(256) k(float *out, const float *win, float wp0, float wp1, float wp2, float wp3,
                                         int iters) {
  float w0, w1, w2, w3;
  if (FORM == 0) { w0 = win[0]; w1 = win[1]; w2 = win[2]; w3 = win[3]; }
  float a[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 1e-3f + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (FORM == 0) a[i] = __fmaf_rn(a[i], w0 + 0.f * i, w1);
      if (FORM == 1) a[i] = __fmaf_rn(a[i], wp0, wp1);
      if (FORM == 2) a[i] = __fmaf_rn(a[i], 0.999f, 0.001f);
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      if (FORM == 0) a[i] = __fmaf_rn(a[i], w2, w3);
      if (FORM == 1) a[i] = __fmaf_rn(a[i], wp2, wp3);
      if (FORM == 2) a[i] = __fmaf_rn(a[i], 0.998f, 0.002f);
    }
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Packed FFMA2 (fma.rn.f32x2, sm_100): 16 pair accumulators = 32 FMA lanes per
// iteration half, same dependency depth as the scalar forms.
__global__ void __launch_bounds__(256) k2(float *out, const float *win, int iters) {
  unsigned long long w01, w23, a[16];
  asm("mov.b64 %0, {%1,%2};" : "=l"(w01) : "f"(win[0]), "f"(win[1]));
  asm("mov.b64 %0, {%1,%2};" : "=l"(w23) : "f"(win[2]), "f"(win[3]));
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const float v = threadIdx.x * 1e-3f + i;
    asm("mov.b64 %0, {%1,%2};" : "=l"(a[i]) : "f"(v), "f"(v + 0.5f));
  }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(w01), "l"(w23));
#pragma unroll
    for (int i = 0; i < 16; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(w23), "l"(w01));
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    float x, y;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(x), "=f"(y) : "l"(a[i]));
    s += x + y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  float *out, *win;
  cudaMalloc(&out, 148 * 8 * 256 * 4);
  cudaMalloc(&win, 16);
  float h[4] = {0.999f, 0.001f, 0.998f, 0.002f};
  cudaMemcpy(win, h, 16, cudaMemcpyHostToDevice);
  const int iters = 20000;
  for (int form = 0; form < 3; ++form) {
    for (int bps = 2; bps <= 8; bps *= 2) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      auto kern = form == 0 ? k<0> : form == 1 ? k<1> : k<2>;
      kern<<<148 * bps, 256>>>(out, win, h[0], h[1], h[2], h[3], 100);
      cudaEventRecord(e0);
      kern<<<148 * bps, 256>>>(out, win, h[0], h[1], h[2], h[3], iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      double fma = 148.0 * bps * 256 * iters * 32;
      printf("form %d (%s) ctas/SM %d: %.2f TFLOP/s fp32\n", form, form == 0 ? "3-reg" : form == 1 ? "param" : "imm",
             bps, 2 * fma / ms / 1e9);
    }
  }
  for (int bps = 2; bps <= 8; bps *= 2) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    k2<<<148 * bps, 256>>>(out, win, 100);
    cudaEventRecord(e0);
    k2<<<148 * bps, 256>>>(out, win, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fma = 148.0 * bps * 256 * iters * 64;
    printf("form 3 (ffma2 packed) ctas/SM %d: %.2f TFLOP/s fp32\n", bps, 2 * fma / ms / 1e9);
  }
  return 0;
}
