// k_matvec.cu -- the MATVEC loop body (the paper's
// fourth evaluation kernel, sizes PAPER.md:1405-1430):
//   y[i] = sum_k A[i][k] * x[k]
// as a worksharing upir.loop over the rows i (reading c29):
//   distribute(teams)      : rows are scheduled over TEAMS; inside a row the
//                            k-loop is a nested worksharing loop over the
//                            team's UNITS (static, inner chunk ic) with a
//                            reduction(+) over the units -- coalesced 16-B
//                            loads of A, x re-read from L1/L2.
//   distribute(teams,units): rows are scheduled over the flat units; each unit
//                            runs its row's k-loop sequentially.
// HBM-bound: 4 B of A per multiply-add.  fp32 loads, fp32 FMA with four
// independent accumulators per unit, fixed-order warp/team tree.
#include "sched.cuh"
#include "upir_internal.h"

namespace upir {
namespace {

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int m = 16; m >= 1; m >>= 1) v += __shfl_xor_sync(0xffffffffu, v, m);
  return v;
}

// Row iterator of the row loop for team t of p (static block / static,c /
// dynamic tickets claimed by thread 0).
struct RowIter {
  int64_t cur, end, k;
  bool started;
};

__device__ __forceinline__ int64_t next_row(RowIter &it, const MatvecArgs &a, int64_t T, int64_t p, int64_t t) {
  if (it.cur < it.end) return it.cur++;
  if (a.sched == SK_STATIC_BLOCK) {
    if (it.started) return -1;
    it.started = true;
    block_range(T, a.simd, p, t, it.cur, it.end);   // groups of a.simd rows (c33)
  } else if (a.sched == SK_STATIC_CHUNK) {
    const int64_t kk = it.started ? it.k + p : t;
    it.started = true;
    it.k = kk;
    it.cur = kk * a.chunk;
    it.end = min(T, it.cur + a.chunk);
  } else {
    const int64_t kk = (int64_t)atomicAdd(a.dyn_counter, 1ull);
    it.cur = kk * a.chunk;
    it.end = min(T, it.cur + a.chunk);
  }
  if (it.cur >= it.end) return -1;
  return it.cur++;
}

// distribute(teams): one team per row at a time, units split the k-loop.
// One barrier per row: the row id of iteration it+1 and the warp partials of
// row it are published together (double-buffered), and warp 0 finishes row
// it's reduction while the team streams row it+1.
__global__ void __launch_bounds__(1024) matvec_teams_kernel(const __grid_constant__ MatvecArgs a) {
  __shared__ float s_part[2][32];
  __shared__ long long s_row[2];
  __shared__ unsigned s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = (blockDim.x + 31) >> 5;
  const int units = blockDim.x, u = threadIdx.x;
  const int64_t T = a.T;
  RowIter it{0, 0, 0, false};
  const bool vec = a.inner_chunk == 4 && (a.lda % 4) == 0 && (((uintptr_t)a.A | (uintptr_t)a.x) % 16) == 0;
  if (threadIdx.x == 0) s_row[0] = next_row(it, a, T, gridDim.x, blockIdx.x);
  __syncthreads();
  int64_t prev = -1;   // row whose partials sit in s_part[(iter - 1) & 1]
  for (int iter = 0;; ++iter) {
    const int buf = iter & 1;
    const int64_t r = s_row[buf];
    // warp 0 finishes the previous row (its partials were published by the last barrier)
    if (prev >= 0 && warp == 0) {
      if (lane == 0) {
        float s = 0.f;
        for (int w = 0; w < nwarps; ++w) s += s_part[buf ^ 1][w];
        a.y[a.lb + prev] = s;
        if (a.trace) {
          a.trace[prev] = blockIdx.x;
          a.trace[T + prev] = 0;
          atomicAdd(a.trace + 2 * T + prev, 1);
        }
      }
      __syncwarp();
    }
    if (r < 0) break;
    const int64_t i = a.lb + r;
    const float *Ai = a.A + i * a.lda;
    float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
    if (vec) {
      // static, 4 over units: chunk c = 4 consecutive k -> unit c mod units
      const int64_t nc = a.K / 4;
      int64_t c = u;
      for (; c + 3 * (int64_t)units < nc; c += 4 * (int64_t)units) {
        float4 av[4], xv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          av[q] = __ldcs(reinterpret_cast<const float4 *>(Ai) + c + q * units);
          xv[q] = __ldg(reinterpret_cast<const float4 *>(a.x) + c + q * units);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc0 = __fmaf_rn(av[q].x, xv[q].x, acc0);
          acc1 = __fmaf_rn(av[q].y, xv[q].y, acc1);
          acc2 = __fmaf_rn(av[q].z, xv[q].z, acc2);
          acc3 = __fmaf_rn(av[q].w, xv[q].w, acc3);
        }
      }
      for (; c < nc; c += units) {
        const float4 av = __ldcs(reinterpret_cast<const float4 *>(Ai) + c);
        const float4 xv = __ldg(reinterpret_cast<const float4 *>(a.x) + c);
        acc0 = __fmaf_rn(av.x, xv.x, acc0);
        acc1 = __fmaf_rn(av.y, xv.y, acc1);
        acc2 = __fmaf_rn(av.z, xv.z, acc2);
        acc3 = __fmaf_rn(av.w, xv.w, acc3);
      }
      // ragged tail of the row (K % 4): chunk nc belongs to unit nc mod units
      if ((a.K & 3) && u == (int)(nc % units))
        for (int64_t k = nc * 4; k < a.K; ++k) acc0 = __fmaf_rn(Ai[k], a.x[k], acc0);
    } else {
      const int64_t ic = a.inner_chunk;
      for (int64_t c = u; c * ic < a.K; c += units)
        for (int64_t k = c * ic; k < min(a.K, c * ic + ic); ++k) acc0 = __fmaf_rn(Ai[k], a.x[k], acc0);
    }
    float v = (acc0 + acc1) + (acc2 + acc3);
    // team reduction(+) in a fixed order (reading c10): warp tree, then warps in order
    const int rem = units & 31;
    if (warp == nwarps - 1 && rem) {
      float s2 = v;
      for (int l = 1; l < rem; ++l) s2 += __shfl_sync((1u << rem) - 1u, v, l);
      v = s2;
    } else {
      v = warp_sum(v);
    }
    if (lane == 0) s_part[buf][warp] = v;
    if (threadIdx.x == 0) s_row[buf ^ 1] = next_row(it, a, T, gridDim.x, blockIdx.x);
    prev = r;
    __syncthreads();
  }
  if (a.sched == SK_DYNAMIC) {
    __syncthreads();
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

// distribute(teams,units): each unit owns whole rows (static schedules).
__global__ void __launch_bounds__(1024) matvec_units_kernel(const __grid_constant__ MatvecArgs a) {
  const int64_t p = (int64_t)gridDim.x * blockDim.x, g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t T = a.T;
  RowIter it{0, 0, 0, false};
  for (int64_t r = next_row(it, a, T, p, g); r >= 0; r = next_row(it, a, T, p, g)) {
    const int64_t i = a.lb + r;
    const float *Ai = a.A + i * a.lda;
    float acc0 = 0.f, acc1 = 0.f;
    int64_t k = 0;
    for (; k + 2 <= a.K; k += 2) {
      acc0 = __fmaf_rn(__ldcs(Ai + k), __ldg(a.x + k), acc0);
      acc1 = __fmaf_rn(__ldcs(Ai + k + 1), __ldg(a.x + k + 1), acc1);
    }
    for (; k < a.K; ++k) acc0 = __fmaf_rn(Ai[k], a.x[k], acc0);
    a.y[i] = acc0 + acc1;
    if (a.trace) {
      a.trace[r] = blockIdx.x;
      a.trace[T + r] = threadIdx.x;
      atomicAdd(a.trace + 2 * T + r, 1);
    }
  }
}

}  // namespace

cudaError_t launch_matvec(const MatvecArgs &a, int teams, int units, cudaStream_t s) {
  if (a.distribute == UPIR_DIST_TEAMS) matvec_teams_kernel<<<teams, units, 0, s>>>(a);
  else matvec_units_kernel<<<teams, units, 0, s>>>(a);
  return cudaGetLastError();
}

}  // namespace upir
