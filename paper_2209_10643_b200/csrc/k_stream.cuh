// k_stream.cuh -- 1-D streaming loop kernels of upir_loop_exec:
//   AXPY   : y[i] = y[i] + a * x[i]            (Fig. 9,
//                                               1180-1186 Fig. 11)
//   REDUCE : private partial p_u = (+)_{i in chunks(u)} x[i]  (Fig. 7 sync
//            'reduction'; [REM] 929-948 mode all-unit)
// run under the device schedule engine (sched.cuh) with the upir.sync
// reduction fused into the loop kernel's end (reduction +
// barrier fusion): warp butterfly -> team -> per-team slot -> last team
// combines the slots in a fixed order and applies init (readings c9, c10).
//
// Two memory paths:
//  DIRECT (default): every unit loads its own elements.  One-vector chunks
//           (chunked static / dynamic with c = one 16-B vector): adjacent
//           units own adjacent vectors, so a warp's loads are coalesced (the
//           x / y of 4 chunks in flight; reductions 6 chunks).  Long chunks (static block, large
//           c): each unit streams its own range with 256-bit loads
//           (ld.global.cs.L2::256B), several in flight; vectors are aligned by
//           ADDRESS (esh), so adopted views with a storage offset and BLOCK
//           slices that start mid-line stay legal.  AXPY teams of <= 256
//           units run the 256-thread compile (no register spills), long
//           chunks with one resident team per SM.
//  STAGED (UPIR_PATH=staged): every unit moves its own next 64-256 B segment
//           into a private shared-memory row with one TMA bulk copy (NST
//           stages deep, mbarrier-tracked) and executes the body on ITS OWN
//           iterations from that row.  AXPY results go back by bulk store,
//           element-exact at unit boundaries.  Kept as the coalesced
//           alternative; measured slower than DIRECT on B200.
#pragma once
#include <cuda_runtime.h>
#include <math_constants.h>
#include <stdint.h>

#include <cstdlib>
#include <type_traits>

#include "dev_peer.cuh"
#include "sched.cuh"

// one-vector-chunk reductions: chunks of a unit in flight (C2, 2^30 int64 /
// fp32 at 592 x 256, measured on B200: 2 / 4 / 5 / 6 / 7 / 8 -> 6.19 / 7.06 /
// 7.09 / 7.20 / 7.16 / 6.98 TB/s per C2 step)
#ifndef UPIR_RED_UF
#define UPIR_RED_UF 6
#endif
// AXPY one-vector chunks (x and y of each): 4 / 6 / 8 in flight -> 0.99-1.00 /
// 0.97 / 0.98 of copy (measured): 4
#ifndef UPIR_AXPY_UF
#define UPIR_AXPY_UF 4
#endif

namespace upir {

static constexpr unsigned FULL = 0xffffffffu;

// ---------------------------------------------------------------- combine ops
__device__ __forceinline__ long long comb_i64(int op, long long a, long long b) {
  if (op == UPIR_OP_SUM) return (long long)((unsigned long long)a + (unsigned long long)b);
  if (op == UPIR_OP_MAX) return a > b ? a : b;
  return a < b ? a : b;
}
__device__ __forceinline__ double comb_f(int op, double a, double b) {
  if (op == UPIR_OP_SUM) return a + b;
  if (op == UPIR_OP_MAX) return fmax(a, b);
  return fmin(a, b);
}
__device__ __forceinline__ long long ident_i64(int op) {
  return op == UPIR_OP_SUM ? 0LL : (op == UPIR_OP_MAX ? (long long)INT64_MIN : (long long)INT64_MAX);
}
__device__ __forceinline__ double ident_f(int op) {
  return op == UPIR_OP_SUM ? 0.0 : (op == UPIR_OP_MAX ? -CUDART_INF : CUDART_INF);
}
__device__ __forceinline__ float ident_f32(int op) {
  return op == UPIR_OP_SUM ? 0.0f : (op == UPIR_OP_MAX ? -CUDART_INF_F : CUDART_INF_F);
}

// Private reduction copies of one unit.  int64 data: exact int64 words.
// fp32 data: fp64 words (reading c11: the private partial of a unit is kept
// in double; each 16-B vector is first combined pairwise in fp32).
template <int BODY, int NRED>
struct Acc {
  using W = typename std::conditional<BODY == SB_RED_I64, long long, double>::type;
  W v[NRED > 0 ? NRED : 1];
  int op[NRED > 0 ? NRED : 1];
  __device__ __forceinline__ void init(const StreamArgs &a) {
#pragma unroll
    for (int r = 0; r < NRED; ++r) {
      op[r] = a.red[r].op;
      if constexpr (BODY == SB_RED_I64) v[r] = ident_i64(op[r]);
      else v[r] = ident_f(op[r]);
    }
  }
};

// ---------------------------------------------------------------- memory ops
__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <bool TRACE>
__device__ __forceinline__ void trace_rec(const StreamArgs &a, int64_t e, int team, int unit) {
  if constexpr (TRACE) {
    const int64_t k = (e - a.lb) / a.step;   // normalised iteration of element e
    a.trace[k] = team;
    a.trace[a.T + k] = unit;
    atomicAdd(a.trace + 2 * a.T + k, 1);
  }
}

// Body on one element (scalar form).
template <int BODY, int NRED, bool TRACE>
__device__ __forceinline__ void body_scalar(const StreamArgs &a, int64_t e, Acc<BODY, NRED> &acc,
                                            int team, int unit) {
  if constexpr (BODY == SB_RED_I64) {
    const long long v = __ldcs(reinterpret_cast<const long long *>(a.in0) + e);
#pragma unroll
    for (int r = 0; r < NRED; ++r) acc.v[r] = comb_i64(acc.op[r], acc.v[r], v);
  } else if constexpr (BODY == SB_RED_F32) {
    const float v = __ldcs(reinterpret_cast<const float *>(a.in0) + e);
#pragma unroll
    for (int r = 0; r < NRED; ++r) acc.v[r] = comb_f(acc.op[r], acc.v[r], (double)v);
  } else {
    const float x = __ldcs(reinterpret_cast<const float *>(a.in0) + e);
    float *yp = reinterpret_cast<float *>(a.out) + e;
    const float y = __ldcs(yp);
    const float yn = __fmaf_rn(a.alpha, x, y);
    __stcs(yp, yn);
#pragma unroll
    for (int r = 0; r < NRED; ++r) acc.v[r] = comb_f(acc.op[r], acc.v[r], (double)yn);
  }
  trace_rec<TRACE>(a, e, team, unit);
}

// Combine a 4-wide fp32 vector into the fp64 partials, masked lanes replaced
// by the identity (pairwise in fp32 first).
template <int BODY, int NRED>
__device__ __forceinline__ void acc_f4(Acc<BODY, NRED> &acc, float4 v, bool m0, bool m1, bool m2,
                                       bool m3) {
#pragma unroll
  for (int r = 0; r < NRED; ++r) {
    const int op = acc.op[r];
    const float id = ident_f32(op);
    const float a0 = m0 ? v.x : id, a1 = m1 ? v.y : id, a2 = m2 ? v.z : id, a3 = m3 ? v.w : id;
    float s;
    if (op == UPIR_OP_SUM) s = __fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3));
    else if (op == UPIR_OP_MAX) s = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3));
    else s = fminf(fminf(a0, a1), fminf(a2, a3));
    acc.v[r] = comb_f(op, acc.v[r], (double)s);
  }
}

template <int BODY, int NRED>
__device__ __forceinline__ void acc_l2(Acc<BODY, NRED> &acc, longlong2 v, bool m0, bool m1) {
#pragma unroll
  for (int r = 0; r < NRED; ++r) {
    const int op = acc.op[r];
    if (m0) acc.v[r] = comb_i64(op, acc.v[r], v.x);
    if (m1) acc.v[r] = comb_i64(op, acc.v[r], v.y);
  }
}

// ================================================================ DIRECT path
template <int BODY, int NRED, bool TRACE>
__device__ __forceinline__ void direct_vec(const StreamArgs &a, int64_t e, Acc<BODY, NRED> &acc,
                                           int team, int unit) {
  // one aligned, full 16-B vector starting at element e
  if constexpr (BODY == SB_RED_I64) {
    const longlong2 v = __ldcs(reinterpret_cast<const longlong2 *>(reinterpret_cast<const long long *>(a.in0) + e));
    acc_l2(acc, v, true, true);
  } else if constexpr (BODY == SB_RED_F32) {
    const float4 v = __ldcs(reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(a.in0) + e));
    acc_f4(acc, v, true, true, true, true);
  } else {
    const float4 x = __ldcs(reinterpret_cast<const float4 *>(reinterpret_cast<const float *>(a.in0) + e));
    float4 *yp = reinterpret_cast<float4 *>(reinterpret_cast<float *>(a.out) + e);
    float4 y = __ldcs(yp);
    y.x = __fmaf_rn(a.alpha, x.x, y.x);
    y.y = __fmaf_rn(a.alpha, x.y, y.y);
    y.z = __fmaf_rn(a.alpha, x.z, y.z);
    y.w = __fmaf_rn(a.alpha, x.w, y.w);
    __stcs(yp, y);
    acc_f4(acc, y, true, true, true, true);
  }
  if constexpr (TRACE) {
    constexpr int VEC = BODY == SB_RED_I64 ? 2 : 4;
#pragma unroll
    for (int q = 0; q < VEC; ++q) trace_rec<TRACE>(a, e + q, team, unit);
  }
}

// One unit's contiguous element range [elo, ehi) of a reduction body: NV
// 16-B vectors per load (NV = 2: 256-bit LDG with a 256-B L2 prefetch), U
// loads in flight.  Scalar head / tail.
// HINT (AXPY only): 0 = streaming loads and stores (.cs); 1 = streaming
// loads, write-back stores (a unit's 32-B sectors of y' stay in L2 until the
// whole line is dirty: no partial-line evictions / DRAM read-modify-write);
// 2 = write-back stores and default-policy loads.
// LINE = 1: the scalar head aligns the main loop to U*32 B (a full line per
// iteration, so every store of the unit completes whole lines).
template <int BODY, int NRED, int NV, int U, int HINT = 0, int LINE = 0>
__device__ __forceinline__ void direct_long(const StreamArgs &a, int64_t elo, int64_t ehi, int64_t vec_hi,
                                            Acc<BODY, NRED> &acc) {
  constexpr int VEC = BODY == SB_RED_I64 ? 2 : 4;
  constexpr int STEP = VEC * NV;   // elements per load
  constexpr int AL = LINE ? STEP * U : STEP;
  int64_t e = elo;
  const int64_t sh = a.esh;   // vectors are aligned by address, not by index
  const int64_t ea = min(ehi, ((elo + sh + AL - 1) / AL) * AL - sh);
  for (; e < ea; ++e) body_scalar<BODY, NRED, false>(a, e, acc, 0, 0);
  const int64_t eb = max(e, (min(ehi, vec_hi) + sh) / STEP * STEP - sh);
  for (; e + U * STEP <= eb; e += U * STEP) {
    if constexpr (BODY == SB_RED_I64) {
      const long long *p = reinterpret_cast<const long long *>(a.in0) + e;
      longlong2 v[U * NV];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        if constexpr (NV == 2)
          asm("ld.global.cs.L2::256B.v4.s64 {%0,%1,%2,%3}, [%4];"
              : "=l"(v[2 * q].x), "=l"(v[2 * q].y), "=l"(v[2 * q + 1].x), "=l"(v[2 * q + 1].y)
              : "l"(p + q * STEP));
        else
          v[q] = __ldcs(reinterpret_cast<const longlong2 *>(p + q * STEP));
      }
#pragma unroll
      for (int q = 0; q < U * NV; ++q) acc_l2(acc, v[q], true, true);
    } else if constexpr (BODY == SB_AXPY) {
      const float *px = reinterpret_cast<const float *>(a.in0) + e;
      float *py = reinterpret_cast<float *>(a.out) + e;
      float4 x[U * NV], y[U * NV];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        if constexpr (NV == 2 && HINT < 2) {
          asm("ld.global.cs.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
              : "=f"(x[2 * q].x), "=f"(x[2 * q].y), "=f"(x[2 * q].z), "=f"(x[2 * q].w), "=f"(x[2 * q + 1].x),
                "=f"(x[2 * q + 1].y), "=f"(x[2 * q + 1].z), "=f"(x[2 * q + 1].w)
              : "l"(px + q * STEP));
          asm volatile("ld.global.cs.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=f"(y[2 * q].x), "=f"(y[2 * q].y), "=f"(y[2 * q].z), "=f"(y[2 * q].w), "=f"(y[2 * q + 1].x),
                         "=f"(y[2 * q + 1].y), "=f"(y[2 * q + 1].z), "=f"(y[2 * q + 1].w)
                       : "l"(py + q * STEP)
                       : "memory");
        } else if constexpr (NV == 2) {
          asm("ld.global.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
              : "=f"(x[2 * q].x), "=f"(x[2 * q].y), "=f"(x[2 * q].z), "=f"(x[2 * q].w), "=f"(x[2 * q + 1].x),
                "=f"(x[2 * q + 1].y), "=f"(x[2 * q + 1].z), "=f"(x[2 * q + 1].w)
              : "l"(px + q * STEP));
          asm volatile("ld.global.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                       : "=f"(y[2 * q].x), "=f"(y[2 * q].y), "=f"(y[2 * q].z), "=f"(y[2 * q].w), "=f"(y[2 * q + 1].x),
                         "=f"(y[2 * q + 1].y), "=f"(y[2 * q + 1].z), "=f"(y[2 * q + 1].w)
                       : "l"(py + q * STEP)
                       : "memory");
        } else {
          x[q] = __ldcs(reinterpret_cast<const float4 *>(px + q * STEP));
          y[q] = __ldcs(reinterpret_cast<const float4 *>(py + q * STEP));
        }
      }
#pragma unroll
      for (int q = 0; q < U * NV; ++q) {
        y[q].x = __fmaf_rn(a.alpha, x[q].x, y[q].x);
        y[q].y = __fmaf_rn(a.alpha, x[q].y, y[q].y);
        y[q].z = __fmaf_rn(a.alpha, x[q].z, y[q].z);
        y[q].w = __fmaf_rn(a.alpha, x[q].w, y[q].w);
        acc_f4(acc, y[q], true, true, true, true);
      }
#pragma unroll
      for (int q = 0; q < U; ++q) {
        if constexpr (NV == 2 && HINT == 0)
          asm volatile("st.global.cs.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(py + q * STEP), "f"(y[2 * q].x),
                       "f"(y[2 * q].y), "f"(y[2 * q].z), "f"(y[2 * q].w), "f"(y[2 * q + 1].x), "f"(y[2 * q + 1].y),
                       "f"(y[2 * q + 1].z), "f"(y[2 * q + 1].w)
                       : "memory");
        else if constexpr (NV == 2)
          asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(py + q * STEP), "f"(y[2 * q].x),
                       "f"(y[2 * q].y), "f"(y[2 * q].z), "f"(y[2 * q].w), "f"(y[2 * q + 1].x), "f"(y[2 * q + 1].y),
                       "f"(y[2 * q + 1].z), "f"(y[2 * q + 1].w)
                       : "memory");
        else
          __stcs(reinterpret_cast<float4 *>(py + q * STEP), y[q]);
      }
    } else {
      const float *p = reinterpret_cast<const float *>(a.in0) + e;
      float4 v[U * NV];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        if constexpr (NV == 2)
          asm("ld.global.cs.L2::256B.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
              : "=f"(v[2 * q].x), "=f"(v[2 * q].y), "=f"(v[2 * q].z), "=f"(v[2 * q].w), "=f"(v[2 * q + 1].x),
                "=f"(v[2 * q + 1].y), "=f"(v[2 * q + 1].z), "=f"(v[2 * q + 1].w)
              : "l"(p + q * STEP));
        else
          v[q] = __ldcs(reinterpret_cast<const float4 *>(p + q * STEP));
      }
#pragma unroll
      for (int q = 0; q < U * NV; ++q) acc_f4(acc, v[q], true, true, true, true);
    }
  }
  for (; e + VEC <= eb; e += VEC) direct_vec<BODY, NRED, false>(a, e, acc, 0, 0);
  for (; e < ehi; ++e) body_scalar<BODY, NRED, false>(a, e, acc, 0, 0);
}

template <int BODY, int NRED, bool TRACE, int LB = 1024>
__device__ void direct_run(const StreamArgs &a, const LaneWork &w, Acc<BODY, NRED> &acc, int team,
                           int unit) {
  if (w.nk == 0) return;
  constexpr int VEC = BODY == SB_RED_I64 ? 2 : 4;
  int64_t j = 0;
  if (a.vecok && a.step == 1 && w.c == VEC && w.nk > 1 && ((a.lb + w.lo0 + a.esh) % VEC) == 0 &&
      (w.kstride % VEC) == 0) {
    // chunks that are one full, aligned vector inside the safe range
    const int64_t lim = min(a.T, a.safe_hi - a.lb);   // need klo + VEC <= lim
    int64_t nfull = 0;
    if (lim - VEC - w.lo0 >= 0) nfull = min(w.nk, (lim - VEC - w.lo0) / w.kstride + 1);
    const int64_t e0 = a.lb + w.lo0;
    // reductions: UF one-vector chunks of the unit in flight (loaded, then
    // combined in chunk order: the unit's partial is the same sequence)
    constexpr int UF = TRACE ? 4 : (BODY == SB_AXPY ? UPIR_AXPY_UF : UPIR_RED_UF);
    for (; j + UF <= nfull; j += UF) {
      if constexpr (BODY == SB_AXPY && !TRACE) {
        // the 4 chunks' x and y vectors are all loaded before any y' store
        // (the chunks are distinct elements, so this holds even when x and y
        // alias): 8 loads in flight per unit instead of 2
        const float *px = reinterpret_cast<const float *>(a.in0);
        float *py = reinterpret_cast<float *>(a.out);
        float4 xv[UF], yv[UF];
#pragma unroll
        for (int q = 0; q < UF; ++q) {
          xv[q] = __ldcs(reinterpret_cast<const float4 *>(px + e0 + (j + q) * w.kstride));
          yv[q] = __ldcs(reinterpret_cast<const float4 *>(py + e0 + (j + q) * w.kstride));
        }
#pragma unroll
        for (int q = 0; q < UF; ++q) {
          yv[q].x = __fmaf_rn(a.alpha, xv[q].x, yv[q].x);
          yv[q].y = __fmaf_rn(a.alpha, xv[q].y, yv[q].y);
          yv[q].z = __fmaf_rn(a.alpha, xv[q].z, yv[q].z);
          yv[q].w = __fmaf_rn(a.alpha, xv[q].w, yv[q].w);
          __stcs(reinterpret_cast<float4 *>(py + e0 + (j + q) * w.kstride), yv[q]);
          acc_f4(acc, yv[q], true, true, true, true);
        }
      } else if constexpr (BODY == SB_AXPY || TRACE) {
#pragma unroll
        for (int q = 0; q < UF; ++q) direct_vec<BODY, NRED, TRACE>(a, e0 + (j + q) * w.kstride, acc, team, unit);
      } else if constexpr (BODY == SB_RED_I64) {
        longlong2 v[UF];
        const long long *p = reinterpret_cast<const long long *>(a.in0);
#pragma unroll
        for (int q = 0; q < UF; ++q) v[q] = __ldcs(reinterpret_cast<const longlong2 *>(p + e0 + (j + q) * w.kstride));
#pragma unroll
        for (int q = 0; q < UF; ++q) acc_l2(acc, v[q], true, true);
      } else {
        float4 v[UF];
        const float *p = reinterpret_cast<const float *>(a.in0);
#pragma unroll
        for (int q = 0; q < UF; ++q) v[q] = __ldcs(reinterpret_cast<const float4 *>(p + e0 + (j + q) * w.kstride));
#pragma unroll
        for (int q = 0; q < UF; ++q) acc_f4(acc, v[q], true, true, true, true);
      }
    }
    for (; j < nfull; ++j) direct_vec<BODY, NRED, TRACE>(a, e0 + j * w.kstride, acc, team, unit);
  }
  // long contiguous chunks (static block / large c) with step 1: every unit
  // streams its own range with wide vector loads, several in flight
  // (adjacent units are far apart, so a warp instruction touches 32 lines;
  // each line is then consumed from L1 by the following loads of the lane).
  if (a.vecok && a.step == 1 && w.c > VEC) {
    const int64_t vec_hi = a.safe_hi;
    for (; j < w.nk; ++j) {
      int64_t klo, khi;
      chunk_bounds(w, j, a.T, klo, khi);
      const int64_t elo = a.lb + klo, ehi = a.lb + khi;
      if constexpr (!TRACE) {
        switch (a.dvar) {
          case 1: direct_long<BODY, NRED, 2, 4>(a, elo, ehi, vec_hi, acc); break;
          case 2: direct_long<BODY, NRED, 2, 2>(a, elo, ehi, vec_hi, acc); break;
          case 3: direct_long<BODY, NRED, 1, 8>(a, elo, ehi, vec_hi, acc); break;
          case 4: direct_long<BODY, NRED, 2, 4, 1>(a, elo, ehi, vec_hi, acc); break;
          case 5: direct_long<BODY, NRED, 2, 4, 2>(a, elo, ehi, vec_hi, acc); break;
          case 6: direct_long<BODY, NRED, 2, 2, 1>(a, elo, ehi, vec_hi, acc); break;
          case 7: direct_long<BODY, NRED, 2, 4, 1, 1>(a, elo, ehi, vec_hi, acc); break;
          case 8: direct_long<BODY, NRED, 2, 4, 0, 1>(a, elo, ehi, vec_hi, acc); break;
          case 9: direct_long<BODY, NRED, 2, 2, 1, 1>(a, elo, ehi, vec_hi, acc); break;
          default: direct_long<BODY, NRED, 1, 4>(a, elo, ehi, vec_hi, acc); break;
        }
        continue;
      }
      int64_t e = elo;
      const int64_t sh = a.esh;
      const int64_t ea = min(ehi, ((elo + sh + VEC - 1) / VEC) * VEC - sh);
      for (; e < ea; ++e) body_scalar<BODY, NRED, TRACE>(a, e, acc, team, unit);
      const int64_t eb = max(e, (min(ehi, vec_hi) + sh) / VEC * VEC - sh);
      for (; e + 4 * VEC <= eb; e += 4 * VEC) {
#pragma unroll
        for (int q = 0; q < 4; ++q) direct_vec<BODY, NRED, TRACE>(a, e + q * VEC, acc, team, unit);
      }
      for (; e + VEC <= eb; e += VEC) direct_vec<BODY, NRED, TRACE>(a, e, acc, team, unit);
      for (; e < ehi; ++e) body_scalar<BODY, NRED, TRACE>(a, e, acc, team, unit);
    }
    return;
  }
  // generic remainder: element by element
  for (; j < w.nk; ++j) {
    int64_t klo, khi;
    chunk_bounds(w, j, a.T, klo, khi);
    for (int64_t k = klo; k < khi; ++k) body_scalar<BODY, NRED, TRACE>(a, a.lb + k * a.step, acc, team, unit);
  }
}

// ================================================================ STAGED path
// Per-unit bulk staging: every unit (lane) streams ITS OWN iterations through
// a private shared-memory row with one TMA bulk copy (cp.async.bulk) per
// segment of up to SEGV 16-B vectors, NST stages deep, completion tracked by
// one mbarrier per warp and stage (32 arrivals + transaction bytes).  Rows
// are padded by 16 B so the lanes' LDS.128 reads are bank-conflict free.
// AXPY results are written back from the row with a bulk store (full
// vectors) and element-exact scalar stores at unit boundaries.
template <int BODY, int SEGV, int NST>
struct StagedLayout {
  static constexpr int ROW = SEGV * 16 + 16;
  static constexpr int NBUF = BODY == SB_AXPY ? 2 : 1;
  static constexpr int STAGE = 32 * ROW * NBUF;
  static constexpr int META = 32 * 16;
  static constexpr int WARP_BYTES = ((NST * (STAGE + META) + 8 * NST + 127) / 128) * 128;
};

__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

template <int BODY, int SEGV, int NST>
__device__ __forceinline__ void staged_init(char *wsm) {
  using L = StagedLayout<BODY, SEGV, NST>;
  unsigned long long *bars = reinterpret_cast<unsigned long long *>(wsm + NST * (L::STAGE + L::META));
  if ((threadIdx.x & 31) == 0)
    for (int i = 0; i < NST; ++i) mbar_init(bars + i, 32);
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  __syncwarp();
}

template <int BODY, int NRED, bool TRACE, int SEGV, int NST>
__device__ void staged_run(const StreamArgs &a, const LaneWork &w, Acc<BODY, NRED> &acc, int team, int unit,
                           char *wsm, int64_t &sglob) {
  using L = StagedLayout<BODY, SEGV, NST>;
  constexpr int VEC = BODY == SB_RED_I64 ? 2 : 4;
  constexpr int LOGV = VEC == 2 ? 1 : 2;
  const int lane = threadIdx.x & 31;
  char *rows = wsm;
  longlong2 *meta = reinterpret_cast<longlong2 *>(wsm + NST * L::STAGE);
  unsigned long long *bars = reinterpret_cast<unsigned long long *>(wsm + NST * (L::STAGE + L::META));
  const char *gx = reinterpret_cast<const char *>(a.in0);
  char *gy = reinterpret_cast<char *>(a.out);
  const int64_t vec_hi = (a.safe_hi / VEC) * VEC;

  int64_t j = 0, e_cur = 0, e_end = 0;
  auto next_interval = [&]() -> bool {
    while (e_cur >= e_end) {
      if (j >= w.nk) return false;
      int64_t klo, khi, elo, ehi;
      chunk_bounds(w, j, a.T, klo, khi);
      ++j;
      elem_bounds(a.lb, a.step, klo, khi, elo, ehi);
      const int64_t stg_hi = min(ehi, vec_hi);
      for (int64_t e = max(elo, stg_hi); e < ehi; ++e) body_scalar<BODY, NRED, TRACE>(a, e, acc, team, unit);
      e_cur = elo;
      e_end = stg_hi;
    }
    return true;
  };

  // stage s -> slot s % NST, mbarrier phase parity (s / NST) & 1
  auto issue = [&](int64_t s) -> bool {
    const int slot = (int)(s % NST);
    longlong2 m = make_longlong2(0, 0);
    int64_t v0 = 0, nv = 0;
    if (next_interval()) {
      v0 = (int64_t)((uint64_t)e_cur >> LOGV);
      const int64_t vseg_end = (v0 & ~(int64_t)(SEGV - 1)) + SEGV;   // segments end on SEGV*16-B boundaries
      const int64_t seg_hi = min(e_end, vseg_end << LOGV);
      nv = (int64_t)(((uint64_t)seg_hi + VEC - 1) >> LOGV) - v0;
      m = make_longlong2(e_cur, seg_hi);
      e_cur = seg_hi;
    }
    meta[slot * 32 + lane] = m;
    unsigned long long *bar = bars + slot;
    char *row = rows + slot * L::STAGE + lane * L::ROW;
    if (nv > 0) {
      fence_proxy_async();   // my earlier generic reads of this row precede the async write
      mbar_arrive_tx(bar, (unsigned)(nv * 16 * L::NBUF));
      bulk_g2s(row, gx + v0 * 16, (unsigned)(nv * 16), bar);
      if constexpr (BODY == SB_AXPY) bulk_g2s(row + 32 * L::ROW, gy + v0 * 16, (unsigned)(nv * 16), bar);
    } else {
      mbar_arrive(bar);
    }
    return __any_sync(FULL, nv > 0);
  };

  auto consume_vec = [&](const char *row, int k, int64_t vb, bool full, const longlong2 &m) {
    if constexpr (BODY == SB_RED_I64) {
      const longlong2 v = *reinterpret_cast<const longlong2 *>(row + k * 16);
      if (full) acc_l2(acc, v, true, true);
      else acc_l2(acc, v, vb >= m.x && vb < m.y, vb + 1 >= m.x && vb + 1 < m.y);
    } else if constexpr (BODY == SB_RED_F32) {
      const float4 v = *reinterpret_cast<const float4 *>(row + k * 16);
      if (full) acc_f4(acc, v, true, true, true, true);
      else acc_f4(acc, v, vb >= m.x && vb < m.y, vb + 1 >= m.x && vb + 1 < m.y, vb + 2 >= m.x && vb + 2 < m.y,
                  vb + 3 >= m.x && vb + 3 < m.y);
    } else {
      const float4 x = *reinterpret_cast<const float4 *>(row + k * 16);
      float4 *yr = reinterpret_cast<float4 *>(const_cast<char *>(row) + 32 * L::ROW + k * 16);
      float4 y = *yr;
      y.x = __fmaf_rn(a.alpha, x.x, y.x);
      y.y = __fmaf_rn(a.alpha, x.y, y.y);
      y.z = __fmaf_rn(a.alpha, x.z, y.z);
      y.w = __fmaf_rn(a.alpha, x.w, y.w);
      *yr = y;
      if (full) acc_f4(acc, y, true, true, true, true);
      else acc_f4(acc, y, vb >= m.x && vb < m.y, vb + 1 >= m.x && vb + 1 < m.y, vb + 2 >= m.x && vb + 2 < m.y,
                  vb + 3 >= m.x && vb + 3 < m.y);
    }
    if constexpr (TRACE) {
#pragma unroll
      for (int q = 0; q < VEC; ++q)
        if (vb + q >= m.x && vb + q < m.y) trace_rec<TRACE>(a, vb + q, team, unit);
    }
  };

  auto consume = [&](int64_t s) {
    const int slot = (int)(s % NST);
    mbar_wait(bars + slot, (unsigned)((s / NST) & 1));
    const longlong2 m = meta[slot * 32 + lane];
    if (m.y <= m.x) return;
    const char *row = rows + slot * L::STAGE + lane * L::ROW;
    const int64_t v0 = (int64_t)((uint64_t)m.x >> LOGV);
    const int nv = (int)((((uint64_t)m.y + VEC - 1) >> LOGV) - v0);
    if (nv == SEGV && m.x == (v0 << LOGV) && m.y == ((v0 + SEGV) << LOGV)) {
#pragma unroll
      for (int k = 0; k < SEGV; ++k) consume_vec(row, k, (v0 + k) << LOGV, true, m);
    } else {
#pragma unroll
      for (int k = 0; k < SEGV; ++k)
        if (k < nv) consume_vec(row, k, (v0 + k) << LOGV, false, m);
    }
    if constexpr (BODY == SB_AXPY) {
      // write back y': full vectors by one bulk store, boundary vectors element-exact
      const float *yrow = reinterpret_cast<const float *>(row + 32 * L::ROW);
      const int64_t f0 = (m.x + VEC - 1) >> LOGV;         // first full vector
      const int64_t f1 = m.y >> LOGV;                      // end of full vectors
      for (int64_t e = m.x; e < min((int64_t)m.y, f0 << LOGV); ++e) reinterpret_cast<float *>(gy)[e] = yrow[e - (v0 << LOGV)];
      if (f1 > f0) {
        fence_proxy_async();   // generic smem writes of y' -> visible to the bulk store
        bulk_s2g(gy + f0 * 16, row + 32 * L::ROW + (f0 - v0) * 16, (unsigned)((f1 - f0) * 16));
        bulk_commit();
      }
      for (int64_t e = max((int64_t)m.x, f1 << LOGV); e < m.y; ++e) reinterpret_cast<float *>(gy)[e] = yrow[e - (v0 << LOGV)];
    }
  };

  int64_t s_issue = sglob, s_cons = sglob;
  bool more = true;
#pragma unroll
  for (int q = 0; q < NST - 1; ++q) {
    if (more) {
      more = issue(s_issue);
      ++s_issue;
    }
  }
  while (s_cons < s_issue) {
    if (more) {
      if constexpr (BODY == SB_AXPY) bulk_wait_read0();   // the slot's last bulk store has read its row
      more = issue(s_issue);
      ++s_issue;
    }
    consume(s_cons);
    ++s_cons;
  }
  if constexpr (BODY == SB_AXPY) bulk_wait0();
  sglob = s_issue;
}

// ================================================================ epilogue
// Team tree then last-team combine (reading c10).  Words are 8 bytes.
template <int BODY, int NRED>
__device__ void reduce_epilogue(const StreamArgs &a, Acc<BODY, NRED> &acc, bool need_ticket) {
  __shared__ unsigned long long s_part[32][2];
  __shared__ int s_last;
  using W = typename Acc<BODY, NRED>::W;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = (blockDim.x + 31) >> 5;
  auto comb = [](int op, W x, W y) -> W {
    if constexpr (BODY == SB_RED_I64) return comb_i64(op, x, y);
    else return comb_f(op, x, y);
  };
  auto ident = [](int op) -> W {
    if constexpr (BODY == SB_RED_I64) return ident_i64(op);
    else return ident_f(op);
  };
  auto to_bits = [](W x) -> unsigned long long {
    if constexpr (BODY == SB_RED_I64) return (unsigned long long)x;
    else return (unsigned long long)__double_as_longlong(x);
  };
  auto from_bits = [](unsigned long long b) -> W {
    if constexpr (BODY == SB_RED_I64) return (W)(long long)b;
    else return __longlong_as_double((long long)b);
  };
  // Warp combine over the wl lanes that exist (a team's last warp may be
  // partial when num_units % 32 != 0): butterfly for full warps, ordered
  // gather to lane 0 otherwise.  Fixed order either way (reading c10).
  auto warp_comb = [&](int op, W x, int wl) -> W {
    if (wl == 32) {
#pragma unroll
      for (int m = 16; m >= 1; m >>= 1) x = comb(op, x, from_bits(__shfl_xor_sync(FULL, to_bits(x), m)));
      return x;
    }
    const unsigned mask = (1u << wl) - 1u;
    W acc = x;
    for (int l = 1; l < wl; ++l) {
      const W o = from_bits(__shfl_sync(mask, to_bits(x), l));
      acc = comb(op, acc, o);
    }
    return acc;   // valid in lane 0
  };
  const int rem = (int)(blockDim.x & 31u);
  const int my_wl = (warp == nwarps - 1 && rem) ? rem : 32;
  const int w0_wl = blockDim.x >= 32 ? 32 : (int)blockDim.x;
  auto block_tree = [&](W (&v)[NRED > 0 ? NRED : 1]) {
#pragma unroll
    for (int r = 0; r < NRED; ++r) {
      v[r] = warp_comb(a.red[r].op, v[r], my_wl);
      if (lane == 0) s_part[warp][r] = to_bits(v[r]);
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
      for (int r = 0; r < NRED; ++r) {
        W x = lane < nwarps ? from_bits(s_part[lane][r]) : ident(a.red[r].op);
        v[r] = warp_comb(a.red[r].op, x, w0_wl);
      }
    }
    __syncthreads();
  };

  if constexpr (NRED > 0) {
    block_tree(acc.v);
    if (threadIdx.x == 0) {
#pragma unroll
      for (int r = 0; r < NRED; ++r) a.slots[(size_t)blockIdx.x * 2 + r] = to_bits(acc.v[r]);
    }
  }
  if (!need_ticket) return;
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned t = atomicAdd(a.done, 1u);
    s_last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if constexpr (NRED > 0) {
    W v[NRED];
#pragma unroll
    for (int r = 0; r < NRED; ++r) {
      W x = ident(a.red[r].op);
      for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x)
        x = comb(a.red[r].op, x, from_bits(__ldcg(a.slots + (size_t)b * 2 + r)));
      v[r] = x;
    }
    block_tree(v);
    if (threadIdx.x == 0 && a.wwin) {
      // upir.sync allreduce fused into the loop's end barrier: publish this
      // rank's partials into every rank's window (slot [parity][rank][r]),
      // signal, wait for all ranks, combine init (+) P_0 (+) ... in ascending
      // rank order.  Parity double-buffering: a rank can only be one world
      // reduction ahead of any other (it waits for all of them each time).
      unsigned long long *win = a.wwin;
      const unsigned long long e = *reinterpret_cast<volatile unsigned long long *>(win + WIN_WR_GEN);
      const int par = (int)(e & 1ull);
      for (int q = 0; q < a.wranks; ++q) {
        unsigned long long *pw = reinterpret_cast<unsigned long long *>(win[WIN_PEERS + q]);
#pragma unroll
        for (int r = 0; r < NRED; ++r)
          st_relaxed_sys(pw + WIN_WR_SLOTS + (par * WIN_MAX_RANKS + a.wrank) * 2 + r, to_bits(v[r]));
      }
      for (int q = 0; q < a.wranks; ++q)
        red_release_sys_add(reinterpret_cast<unsigned long long *>(win[WIN_PEERS + q]) + WIN_WR_CNT, 1ull);
      wait_geq_sys(win + WIN_WR_CNT, (e + 1ull) * (unsigned long long)a.wranks);
#pragma unroll
      for (int r = 0; r < NRED; ++r) {
        const RedSpec &rs = a.red[r];
        W x = from_bits(rs.init_bits);
        for (int q = 0; q < a.wranks; ++q)
          x = comb(rs.op, x, from_bits(ld_relaxed_sys(win + WIN_WR_SLOTS + (par * WIN_MAX_RANKS + q) * 2 + r)));
        if constexpr (BODY == SB_RED_I64) *reinterpret_cast<long long *>(rs.result) = x;
        else *reinterpret_cast<float *>(rs.result) = (float)x;
      }
      *reinterpret_cast<volatile unsigned long long *>(win + WIN_WR_GEN) = e + 1ull;
    } else if (threadIdx.x == 0 && a.wpart) {
#pragma unroll
      for (int r = 0; r < NRED; ++r) a.wpart[r] = to_bits(v[r]);   // combined over ranks by the host path
    } else if (threadIdx.x == 0) {
#pragma unroll
      for (int r = 0; r < NRED; ++r) {
        const RedSpec &rs = a.red[r];
        if constexpr (BODY == SB_RED_I64) {
          const long long res = comb_i64(rs.op, (long long)rs.init_bits, v[r]);
          *reinterpret_cast<long long *>(rs.result) = res;
        } else {
          const double res = comb_f(rs.op, __longlong_as_double((long long)rs.init_bits), v[r]);
          *reinterpret_cast<float *>(rs.result) = (float)res;
        }
      }
    }
  }
  if (threadIdx.x == 0) {
    *a.done = 0u;                                      // self-reset for the next launch
    if (a.dyn_counter) *a.dyn_counter = 0ull;
  }
}

// ================================================================ kernel
template <int BODY, int NRED, bool TRACE, int PATH, int SEGV, int NST, int LB = 1024>
__global__ void __launch_bounds__(LB, LB <= 256 ? 2 : 1) stream_loop_kernel(const __grid_constant__ StreamArgs a) {
  extern __shared__ __align__(128) char dyn_smem[];
  const UnitIds u = unit_ids(a.distribute);
  const int team = blockIdx.x, unit = threadIdx.x;
  Acc<BODY, NRED> acc;
  acc.init(a);
  char *wsm = nullptr;
  int64_t sglob = 0;   // staged: stage counter of this warp (mbarrier phases)
  if constexpr (PATH == PATH_STAGED) {
    wsm = dyn_smem + (threadIdx.x >> 5) * StagedLayout<BODY, SEGV, NST>::WARP_BYTES;
    staged_init<BODY, SEGV, NST>(wsm);
  }

  auto run = [&](const LaneWork &w) {
    if constexpr (PATH == PATH_STAGED) staged_run<BODY, NRED, TRACE, SEGV, NST>(a, w, acc, team, unit, wsm, sglob);
    else direct_run<BODY, NRED, TRACE, LB>(a, w, acc, team, unit);
  };

  if (a.sched == SK_DYNAMIC || a.sched == SK_GUIDED) {
    __shared__ long long s_base;
    const bool guided = a.sched == SK_GUIDED;
    const int64_t nchunks = guided ? a.gchunks : (a.T + a.chunk - 1) / a.chunk;
    const unsigned long long tu = (unsigned long long)u.p_team * (unsigned long long)(guided ? 1 : a.ticket_m);
    for (;;) {
      if (threadIdx.x == 0) s_base = (long long)atomicAdd(a.dyn_counter, tu);
      __syncthreads();
      const int64_t b = s_base;
      __syncthreads();
      if (b >= nchunks) break;
      run(guided ? guided_work(b, nchunks, a.gtab, u) : ticket_work(b, a.ticket_m, a.T, a.chunk, u));
    }
  } else {
    run(static_work(a.sched, a.T, a.chunk, u, a.simd));
  }
  reduce_epilogue<BODY, NRED>(a, acc, NRED > 0 || a.sched == SK_DYNAMIC || a.sched == SK_GUIDED);
}

// Host-side dispatch over (NRED, TRACE, PATH config) for one body.
template <int BODY>
cudaError_t launch_stream_body(int nred, int path, int segv, int nst, bool trace, int teams,
                               int units, size_t smem, const StreamArgs &a, cudaStream_t s) {
  void (*k)(StreamArgs) = nullptr;
#define UPIR_PICK(NR, TR)                                                                  \
  if (path == PATH_DIRECT) k = stream_loop_kernel<BODY, NR, TR, PATH_DIRECT, 0, 0>;          \
  else if (segv == 16 && nst == 3) k = stream_loop_kernel<BODY, NR, TR, PATH_STAGED, 16, 3>; \
  else if (segv == 16 && nst == 2) k = stream_loop_kernel<BODY, NR, TR, PATH_STAGED, 16, 2>; \
  else if (segv == 8 && nst == 3) k = stream_loop_kernel<BODY, NR, TR, PATH_STAGED, 8, 3>;   \
  else if (segv == 8 && nst == 2) k = stream_loop_kernel<BODY, NR, TR, PATH_STAGED, 8, 2>;   \
  else if (segv == 4 && nst == 2) k = stream_loop_kernel<BODY, NR, TR, PATH_STAGED, 4, 2>;
  if (nred == 0) {
    if (trace) { UPIR_PICK(0, true) } else { UPIR_PICK(0, false) }
  } else if (nred == 1) {
    if (trace) { UPIR_PICK(1, true) } else { UPIR_PICK(1, false) }
  } else {
    if (trace) { UPIR_PICK(2, true) } else { UPIR_PICK(2, false) }
  }
#undef UPIR_PICK
  // teams of <= 256 units: the direct kernel compiled for 256 threads (up to
  // 255 registers: the AXPY long-chunk loop keeps 4 x 2 x 32 B of x / y in
  // flight per unit without spilling, which the 64-register bound of a
  // 1024-thread compile cannot)
  // (AXPY by default; experiment hook UPIR_LB256 = 0 never / 1 every body)
  const int lb256 = getenv("UPIR_LB256") ? atoi(getenv("UPIR_LB256")) : -1;
  if (path == PATH_DIRECT && !trace && units <= 256 && (lb256 == 1 || (lb256 < 0 && BODY == SB_AXPY)))
    k = nred == 0 ? stream_loop_kernel<BODY, 0, false, PATH_DIRECT, 0, 0, 256>
        : nred == 1 ? stream_loop_kernel<BODY, 1, false, PATH_DIRECT, 0, 0, 256>
                    : stream_loop_kernel<BODY, 2, false, PATH_DIRECT, 0, 0, 256>;
  if (!k) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k<<<teams, units, smem, s>>>(a);
  return cudaGetLastError();
}

template <int BODY>
size_t staged_bytes_body(int units, int segv, int nst) {
  const int warps = (units + 31) / 32;
  size_t per = 0;
  if (segv == 16 && nst == 3) per = StagedLayout<BODY, 16, 3>::WARP_BYTES;
  else if (segv == 16 && nst == 2) per = StagedLayout<BODY, 16, 2>::WARP_BYTES;
  else if (segv == 8 && nst == 3) per = StagedLayout<BODY, 8, 3>::WARP_BYTES;
  else if (segv == 8 && nst == 2) per = StagedLayout<BODY, 8, 2>::WARP_BYTES;
  else if (segv == 4 && nst == 2) per = StagedLayout<BODY, 4, 2>::WARP_BYTES;
  return per * warps;
}

}  // namespace upir
