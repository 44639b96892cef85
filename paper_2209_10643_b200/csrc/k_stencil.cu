// k_stencil.cu -- the STENCIL2D loop body (the paper's
// "2D stencil, filter size = 7"; reading c28):
//   out[i][j] = sum_{a,b in [-R,R]} w[a+R][b+R] * in[i+a][j+b]
// over a tiled collapse(2) upir.loop (reading c24: tiles anchored at 0, tile
// loop over TEAMS, box positions static,ic over UNITS).  Each team stages the
// (BM+2R) x (BN+2R) input window of its tile in shared memory with coalesced
// loads (rows of the window are contiguous in HBM), the F x F weights once per
// kernel; each unit produces 4 consecutive outputs per chunk from registers
// (register-blocked taps, fp32 FMA in the fixed order of the filter rows /
// columns).  49 FMAs per point at F = 7: ALU-bound rather than HBM-bound.
#include "upir_internal.h"

namespace upir {
namespace {

template <int R, int BM, int BN>
__global__ void __launch_bounds__(1024) stencil_kernel(const __grid_constant__ StencilArgs a) {
  constexpr int F = 2 * R + 1, WR = BM + 2 * R, WC = BN + 2 * R, WCP = WC + 1;
  extern __shared__ float sm[];
  float *win = sm;              // WR x WCP
  float *w = sm + WR * WCP;     // F x F
  __shared__ long long s_tile;
  __shared__ unsigned s_last;
  const int units = blockDim.x, u = threadIdx.x;
  for (int e = threadIdx.x; e < F * F; e += blockDim.x) w[e] = a.w[e];
  const int64_t nt = a.ntr * a.ntc;
  // tile iterator (thread 0), as the Jacobi body
  int64_t cur = 0, end = 0, kk = 0;
  bool started = false;
  auto next_tile = [&]() -> int64_t {
    const int64_t p = gridDim.x, t = blockIdx.x;
    if (cur < end) return cur++;
    if (a.sched == SK_STATIC_BLOCK) {
      if (started) return -1;
      started = true;
      const int64_t q = nt / p, r = nt % p;
      cur = t * q + (t < r ? t : r);
      end = cur + q + (t < r ? 1 : 0);
    } else if (a.sched == SK_STATIC_CHUNK) {
      kk = started ? kk + p : t;
      started = true;
      cur = kk * a.chunk;
      end = min(nt, cur + a.chunk);
    } else {
      kk = (int64_t)atomicAdd(a.dyn_counter, 1ull);
      cur = kk * a.chunk;
      end = min(nt, cur + a.chunk);
    }
    if (cur >= end) return -1;
    return cur++;
  };
  constexpr int POS = BM * BN;
  for (;;) {
    if (threadIdx.x == 0) s_tile = next_tile();
    __syncthreads();
    const int64_t tile = s_tile;
    if (tile < 0) break;
    const int64_t i0 = (a.ti0 + tile / a.ntc) * BM, j0 = (a.tj0 + tile % a.ntc) * BN;
    // stage the window rows [i0-R, i0+BM+R) x cols [j0-R, j0+BN+R)
    for (int e = threadIdx.x; e < WR * WC; e += units) {
      const int r = e / WC, c = e % WC;
      const int64_t gi = i0 - R + r, gj = j0 - R + c;
      float v = 0.f;
      if (gi >= a.row0 && gi < a.ny && gj >= 0 && gj < a.nx) v = __ldcs(a.in + (gi - a.row0) * a.ld + gj);
      win[r * WCP + c] = v;
    }
    __syncthreads();
    const int ic = a.inner_chunk;
    if (ic == 4) {
      for (int k = u; k * 4 < POS; k += units) {
        const int r = (k * 4) / BN, c = (k * 4) % BN;
        const int64_t i = i0 + r, j = j0 + c;
        if (i < a.lb0 || i >= a.ub0 || j + 3 < a.lb1 || j >= a.ub1) continue;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int p = 0; p < F; ++p) {
          float v[4 + 2 * R];
#pragma unroll
          for (int q = 0; q < 4 + 2 * R; ++q) v[q] = win[(r + p) * WCP + c + q];
#pragma unroll
          for (int q = 0; q < F; ++q) {
            const float wq = w[p * F + q];
#pragma unroll
            for (int t = 0; t < 4; ++t) acc[t] = __fmaf_rn(wq, v[t + q], acc[t]);
          }
        }
        float *dst = a.out + (i - a.row0) * a.ld + j;
        if (j >= a.lb1 && j + 4 <= a.ub1 && ((uintptr_t)dst & 15) == 0) {
          __stcs(reinterpret_cast<float4 *>(dst), make_float4(acc[0], acc[1], acc[2], acc[3]));
        } else {
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (j + t >= a.lb1 && j + t < a.ub1) dst[t] = acc[t];
        }
        if (a.trace) {
#pragma unroll
          for (int t = 0; t < 4; ++t)
            if (j + t >= a.lb1 && j + t < a.ub1) {
              const int64_t idx = tile * POS + r * BN + c + t;
              a.trace[idx] = blockIdx.x;
              a.trace[nt * POS + idx] = u;
              atomicAdd(a.trace + 2 * nt * POS + idx, 1);
            }
        }
      }
    } else {
      for (int64_t k = u; k * ic < POS; k += units) {
        for (int pos = (int)(k * ic); pos < (int)min((int64_t)POS, (k + 1) * ic); ++pos) {
          const int r = pos / BN, c = pos % BN;
          const int64_t i = i0 + r, j = j0 + c;
          if (i < a.lb0 || i >= a.ub0 || j < a.lb1 || j >= a.ub1) continue;
          float acc = 0.f;
          for (int p = 0; p < F; ++p)
            for (int q = 0; q < F; ++q) acc = __fmaf_rn(w[p * F + q], win[(r + p) * WCP + c + q], acc);
          a.out[(i - a.row0) * a.ld + j] = acc;
          if (a.trace) {
            const int64_t idx = tile * POS + pos;
            a.trace[idx] = blockIdx.x;
            a.trace[nt * POS + idx] = u;
            atomicAdd(a.trace + 2 * nt * POS + idx, 1);
          }
        }
      }
    }
    __syncthreads();
  }
  if (a.sched == SK_DYNAMIC) {
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(a.done, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && threadIdx.x == 0) {
      *a.done = 0u;
      *a.dyn_counter = 0ull;
    }
  }
}

template <int R, int BM, int BN>
cudaError_t launch_r(const StencilArgs &a, int teams, int units, cudaStream_t s) {
  constexpr int WR = BM + 2 * R, WC = BN + 2 * R + 1, F = 2 * R + 1;
  const size_t smem = (size_t)(WR * WC + F * F) * sizeof(float);
  stencil_kernel<R, BM, BN><<<teams, units, smem, s>>>(a);
  return cudaGetLastError();
}

}  // namespace

bool stencil_supported(int F, int bm, int bn) {
  return (F == 3 || F == 5 || F == 7) && ((bm == 16 && bn == 128) || (bm == 8 && bn == 64));
}

cudaError_t launch_stencil(const StencilArgs &a, int F, int bm, int bn, int teams, int units, cudaStream_t s) {
#define UPIR_ST(R_, BM_, BN_) \
  if (F == 2 * R_ + 1 && bm == BM_ && bn == BN_) return launch_r<R_, BM_, BN_>(a, teams, units, s);
  UPIR_ST(1, 16, 128)
  UPIR_ST(2, 16, 128)
  UPIR_ST(3, 16, 128)
  UPIR_ST(1, 8, 64)
  UPIR_ST(2, 8, 64)
  UPIR_ST(3, 8, 64)
#undef UPIR_ST
  return cudaErrorInvalidValue;
}

}  // namespace upir
