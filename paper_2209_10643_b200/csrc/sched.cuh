// sched.cuh -- device schedule engine of upir.loop_parallel worksharing
// (Fig. 3; readings c3-c8 of DESIGN.md).
//
// A unit's share of the normalised iteration space [0, T) is described as a
// strided sequence of chunks:
//     chunk j = [lo0 + j*kstride, min(lo0 + j*kstride + c, T)),  j in [0, nk)
// static block  : one chunk [g*q + min(g,r), +q + (g<r))
// static chunk c: chunks k = g, g+p, ...   -> lo0 = g*c, kstride = p*c
// dynamic c     : a team claims a ticket of p_team*m consecutive chunks with one
//                 atomicAdd; unit u of the team takes chunks b + u + j*p_team
//                 (j < m): chunk boundaries are exact, each unit's chunks are
//                 increasing, the unit assignment is decided at run time (c8).
// guided c      : the same tickets (m = 1) over the guided chunk sequence
//                 b_{g+1} = b_g + max(ceil((T - b_g)/p), c), precomputed on the
//                 host into a boundary table.
#pragma once
#include <stdint.h>

#include "upir_internal.h"

namespace upir {

struct LaneWork {
  int64_t lo0, kstride, nk, c;
  const int64_t *tab;   // guided: lo0 / kstride index chunks of this boundary table
};

struct UnitIds {
  int64_t g;       // schedule unit id (meaningful when active)
  int64_t p;       // number of schedule units
  int p_team;      // active units in this team (dynamic tickets)
  int u_team;      // index of this unit among the team's active units
  bool active;
};

// distribute (readings c5-c7):
//   TEAMS_UNITS: flat g = team*units + unit, p = teams*units
//   TEAMS      : p = teams, unit 0 of each team executes
//   UNITS      : p = units (a single team)
__device__ __forceinline__ UnitIds unit_ids(int distribute) {
  UnitIds u;
  if (distribute == UPIR_DIST_TEAMS) {
    u.g = blockIdx.x;
    u.p = gridDim.x;
    u.p_team = 1;
    u.u_team = 0;
    u.active = threadIdx.x == 0;
  } else if (distribute == UPIR_DIST_UNITS) {
    u.g = threadIdx.x;
    u.p = blockDim.x;
    u.p_team = blockDim.x;
    u.u_team = threadIdx.x;
    u.active = true;
  } else {
    u.g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    u.p = (int64_t)gridDim.x * blockDim.x;
    u.p_team = blockDim.x;
    u.u_team = threadIdx.x;
    u.active = true;
  }
  return u;
}

// Static block over SIMD groups of s iterations (simdlen, reading c33):
// unit g owns groups [g*q + min(g,r), +q + (g<r)) of G = ceil(T/s); s = 1 is
// the plain block rule.  Returns [start, end) in iterations.
__device__ __forceinline__ void block_range(int64_t T, int64_t s, int64_t p, int64_t g, int64_t &start,
                                            int64_t &end) {
  const int64_t G = s > 1 ? (T + s - 1) / s : T;
  const int64_t q = G / p, r = G % p;
  const int64_t g0 = g * q + (g < r ? g : r);
  const int64_t g1 = g0 + q + (g < r ? 1 : 0);
  start = s > 1 ? g0 * s : g0;
  end = s > 1 ? (g1 * s < T ? g1 * s : T) : g1;
  if (end < start) end = start;
}

__device__ __forceinline__ LaneWork static_work(int sched, int64_t T, int64_t c, const UnitIds &u, int64_t s = 1) {
  LaneWork w{0, 0, 0, 1, nullptr};
  if (!u.active || T <= 0) return w;
  if (sched == SK_STATIC_BLOCK) {
    int64_t start, end;
    block_range(T, s, u.p, u.g, start, end);
    const int64_t len = end - start;
    w.lo0 = start;
    w.c = len > 0 ? len : 1;
    w.nk = len > 0 ? 1 : 0;
    return w;
  }
  // static, chunk c
  const int64_t nchunks = (T + c - 1) / c;
  w.c = c;
  w.lo0 = u.g * c;
  w.kstride = u.p * c;
  w.nk = u.g < nchunks ? (nchunks - 1 - u.g) / u.p + 1 : 0;
  return w;
}

// Unit's chunks of a dynamic ticket starting at chunk b (m chunks per unit).
__device__ __forceinline__ LaneWork ticket_work(int64_t b, int64_t m, int64_t T, int64_t c,
                                                const UnitIds &u) {
  LaneWork w{0, 0, 0, c, nullptr};
  if (!u.active) return w;
  const int64_t nchunks = (T + c - 1) / c;
  const int64_t first = b + u.u_team;
  if (first >= nchunks) return w;
  const int64_t cnt = (nchunks - 1 - first) / u.p_team + 1;
  w.nk = cnt < m ? cnt : m;
  w.lo0 = first * c;
  w.kstride = (int64_t)u.p_team * c;
  return w;
}

// guided: the unit's chunks of a ticket starting at chunk index b of the
// boundary table (chunk g = [tab[g], tab[g+1])); chunk sizes vary, so the
// long-chunk memory paths are used (c = "long").
__device__ __forceinline__ LaneWork guided_work(int64_t b, int64_t nc, const int64_t *tab, const UnitIds &u) {
  LaneWork w{0, 0, 0, ((int64_t)1 << 40), tab};
  if (!u.active) return w;
  const int64_t first = b + u.u_team;
  if (first >= nc) return w;
  w.nk = 1;
  w.lo0 = first;
  return w;
}

// Chunk j of a lane's work, in the normalised space.
__device__ __forceinline__ void chunk_bounds(const LaneWork &w, int64_t j, int64_t T, int64_t &klo,
                                             int64_t &khi) {
  if (w.tab) {
    const int64_t g = w.lo0 + j * w.kstride;
    klo = w.tab[g];
    khi = w.tab[g + 1];
    return;
  }
  klo = w.lo0 + j * w.kstride;
  khi = klo + w.c;
  if (khi > T) khi = T;
}

// Element interval [elo, ehi) covered by normalised [klo, khi) when |step| == 1.
__device__ __forceinline__ void elem_bounds(int64_t lb, int64_t step, int64_t klo, int64_t khi,
                                            int64_t &elo, int64_t &ehi) {
  if (step == 1) {
    elo = lb + klo;
    ehi = lb + khi;
  } else {  // step == -1: i = lb - k
    elo = lb - khi + 1;
    ehi = lb - klo + 1;
  }
}

}  // namespace upir
