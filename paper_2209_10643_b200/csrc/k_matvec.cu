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
// independent accumulators per unit and row, fixed-order warp/team tree.
#include "sched.cuh"
#include "upir_internal.h"

// chunks per unit and row in flight in the two-row k-loop (2 x 4 A vectors +
// 4 x vectors per unit; measured at 16384^2: 2 / 3 / 4 / 5 / 6 -> 0.92 /
// 0.98 / 0.99 / 0.97 / 0.94 of the copy bandwidth, one row at a time 0.95)
constexpr int MV_Q = 4;

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

// A-row loads: streaming, with a 256-B L2 fetch granule (the row is read
// exactly once, in whole 512-B warp spans)
__device__ __forceinline__ float4 ld_a(const float4 *p) {
  float4 v;
  asm volatile("ld.global.cs.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "l"(p));
  return v;
}

// One row's k-loop of unit u (static, inner chunk ic over the team's units)
// into four partial sums, in the unit's fixed order.
struct RowAcc {
  float a0, a1, a2, a3;
  __device__ __forceinline__ void fma4(const float4 &av, const float4 &xv) {
    a0 = __fmaf_rn(av.x, xv.x, a0);
    a1 = __fmaf_rn(av.y, xv.y, a1);
    a2 = __fmaf_rn(av.z, xv.z, a2);
    a3 = __fmaf_rn(av.w, xv.w, a3);
  }
  __device__ __forceinline__ float sum() const { return (a0 + a1) + (a2 + a3); }
};

// distribute(teams): the team takes the rows the schedule hands it two at a
// time (consecutive rows of its sequence; a row never changes team), and its
// units split every row's k-loop.  Both rows stream together: each unit's x
// chunk is loaded once for the pair, and one barrier serves two rows.  The
// row ids of iteration it+1 and the warp partials of iteration it are
// published together (double-buffered); warp 0 finishes iteration it's
// reductions while the team streams iteration it+1.
__global__ void __launch_bounds__(1024) matvec_teams_kernel(const __grid_constant__ MatvecArgs a) {
  __shared__ float s_part[2][2][32];
  __shared__ long long s_row[2][2];
  __shared__ unsigned s_last;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = (blockDim.x + 31) >> 5;
  const int units = blockDim.x, u = threadIdx.x;
  const int64_t T = a.T;
  RowIter it{0, 0, 0, false};
  const bool vec = a.inner_chunk == 4 && (a.lda % 4) == 0 && (((uintptr_t)a.A | (uintptr_t)a.x) % 16) == 0;
  auto claim = [&](int b) {   // thread 0: the next two rows of this team's sequence
    const int64_t r0 = next_row(it, a, T, gridDim.x, blockIdx.x);
    s_row[b][0] = r0;
    s_row[b][1] = r0 >= 0 ? next_row(it, a, T, gridDim.x, blockIdx.x) : -1;
  };
  if (threadIdx.x == 0) claim(0);
  __syncthreads();
  int64_t prev[2] = {-1, -1};   // rows whose partials sit in s_part[(iter - 1) & 1]
  for (int iter = 0;; ++iter) {
    const int buf = iter & 1;
    const int64_t r0 = s_row[buf][0], r1 = s_row[buf][1];
    // warp 0 finishes the previous rows (their partials were published by the last barrier)
    if (prev[0] >= 0 && warp == 0) {
      if (lane < 2 && prev[lane] >= 0) {
        float s = 0.f;
        for (int w = 0; w < nwarps; ++w) s += s_part[buf ^ 1][lane][w];
        a.y[a.lb + prev[lane]] = s;
        if (a.trace) {
          a.trace[prev[lane]] = blockIdx.x;
          a.trace[T + prev[lane]] = 0;
          atomicAdd(a.trace + 2 * T + prev[lane], 1);
        }
      }
      __syncwarp();
    }
    if (r0 < 0) break;
    const float *A0 = a.A + (a.lb + r0) * a.lda;
    const float *A1 = a.A + (a.lb + (r1 >= 0 ? r1 : r0)) * a.lda;   // a lone last row streams once
    RowAcc q0{0.f, 0.f, 0.f, 0.f}, q1{0.f, 0.f, 0.f, 0.f};
    if (vec) {
      // static, 4 over units: chunk c = 4 consecutive k -> unit c mod units
      const int64_t nc = a.K / 4;
      const float4 *X = reinterpret_cast<const float4 *>(a.x);
      const float4 *P0 = reinterpret_cast<const float4 *>(A0), *P1 = reinterpret_cast<const float4 *>(A1);
      int64_t c = u;
      if (r1 >= 0) {
        for (; c + (MV_Q - 1) * (int64_t)units < nc; c += MV_Q * (int64_t)units) {
          float4 a0v[MV_Q], a1v[MV_Q], xv[MV_Q];
#pragma unroll
          for (int q = 0; q < MV_Q; ++q) {
            a0v[q] = ld_a(P0 + c + q * units);
            a1v[q] = ld_a(P1 + c + q * units);
            xv[q] = __ldg(X + c + q * units);
          }
#pragma unroll
          for (int q = 0; q < MV_Q; ++q) {
            q0.fma4(a0v[q], xv[q]);
            q1.fma4(a1v[q], xv[q]);
          }
        }
        for (; c < nc; c += units) {
          const float4 xv = __ldg(X + c);
          q0.fma4(ld_a(P0 + c), xv);
          q1.fma4(ld_a(P1 + c), xv);
        }
      } else {
        for (; c + 3 * (int64_t)units < nc; c += 4 * (int64_t)units) {
          float4 av[4], xv[4];
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            av[q] = ld_a(P0 + c + q * units);
            xv[q] = __ldg(X + c + q * units);
          }
#pragma unroll
          for (int q = 0; q < 4; ++q) q0.fma4(av[q], xv[q]);
        }
        for (; c < nc; c += units) q0.fma4(ld_a(P0 + c), __ldg(X + c));
      }
      // ragged tail of the row (K % 4): chunk nc belongs to unit nc mod units
      if ((a.K & 3) && u == (int)(nc % units))
        for (int64_t k = nc * 4; k < a.K; ++k) {
          q0.a0 = __fmaf_rn(A0[k], a.x[k], q0.a0);
          q1.a0 = __fmaf_rn(A1[k], a.x[k], q1.a0);
        }
    } else {
      const int64_t ic = a.inner_chunk;
      for (int64_t c = u; c * ic < a.K; c += units)
        for (int64_t k = c * ic; k < min(a.K, c * ic + ic); ++k) {
          q0.a0 = __fmaf_rn(A0[k], a.x[k], q0.a0);
          if (r1 >= 0) q1.a0 = __fmaf_rn(A1[k], a.x[k], q1.a0);
        }
    }
    // team reduction(+) per row in a fixed order (reading c10): warp tree,
    // then the warps in order
    float v[2] = {q0.sum(), q1.sum()};
    const int rem = units & 31;
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      if (warp == nwarps - 1 && rem) {
        float s2 = v[e];
        for (int l = 1; l < rem; ++l) s2 += __shfl_sync((1u << rem) - 1u, v[e], l);
        v[e] = s2;
      } else {
        v[e] = warp_sum(v[e]);
      }
    }
    if (lane == 0) {
      s_part[buf][0][warp] = v[0];
      s_part[buf][1][warp] = v[1];
    }
    if (threadIdx.x == 0) claim(buf ^ 1);
    prev[0] = r0;
    prev[1] = r1;
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
