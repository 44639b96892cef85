// k_jacobi.cu -- the JACOBI5 loop body (north_star; reading c16):
//   out[i][j] = 0.25 * ((in[i-1][j] + in[i+1][j]) + (in[i][j-1] + in[i][j+1]))
// over a tiled collapse(2) upir.loop (tiling before
// parallelisation; reading c24).  Tile loop over TEAMS under the loop's
// schedule (static block / static,c / dynamic); inside a tile the BM x BN box
// positions are scheduled static,ic over UNITS.
//
// B200 design: each team (CTA) walks its tiles through an NST-slot ring of
// windows -- the tile's (BM+2) x BN centre box and two (BM+2) x 4 halo-column
// boxes (cp.async.bulk.tensor.2d, mbarrier complete_tx; out-of-range rows /
// columns are zero-filled by the TMA unit and never written).  A dedicated
// producer warp (it executes no iterations, reading c34) claims the tiles in
// schedule order, computes each origin once and refills a slot as soon as
// every unit thread has released it (per-thread arrivals on the slot's empty
// mbarrier); unit warps wait only on their slot's full barrier, never on a
// CTA-wide barrier.  Interior tiles take a lean path (int32 tile-relative
// indexing, west / east neighbours by warp shuffle).  Results are stored as
// coalesced 16-B vectors.  Every input element is read from HBM about once
// per sweep (neighbour tiles' halos hit L2): 8 B per lattice update.
// fp32 arithmetic with explicit __fadd_rn/__fmul_rn: no FMA contraction, so
// the result is independent of decomposition (1 vs N GPUs bit-identical).
//
// Peer mode (a.win != null): the halo exchange with ranks r+-1
// is fused into the sweep.  A unit that computes my first / last owned row
// also stores it into the neighbour's halo row of ITS output buffer (peer
// stores over NVLink), and the tiles that read my halo rows or write those
// boundary rows wait -- before their TMA load is issued -- until both
// neighbours have delivered every sweep before this one (their last team
// bumps my counter with a .sys release after the whole sweep).  Interior
// tiles never wait: the transfer and the neighbour skew overlap the bulk of
// the sweep.
#include <cstdlib>

#include "dev_peer.cuh"
#include "dev_tma.cuh"
#include "upir_internal.h"

namespace upir {

bool encode_tmap_2d(CUtensorMap *out, CUtensorMapDataType dt, const void *base, uint64_t cols, uint64_t rows,
                    uint64_t pitch_bytes, uint32_t box_cols, uint32_t box_rows, CUtensorMapSwizzle swz,
                    CUtensorMapL2promotion l2) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !p)
      return false;
    fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {pitch_bytes};
  cuuint32_t box[2] = {box_cols, box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(out, dt, 2, const_cast<void *>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, swz, l2,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {

constexpr int align128(int x) { return (x + 127) / 128 * 128; }

template <int BM, int BN, int NST>
struct JLayout {
  static constexpr int R = BM + 2;
  static constexpr int CEN = align128(R * BN * 4);
  static constexpr int HAL = align128(R * 4 * 4);
  static constexpr int BUF = CEN + 2 * HAL;
  static constexpr int TX = R * BN * 4 + 2 * R * 16;   // bytes per tile load
  static constexpr int SMEM = NST * BUF + 256;         // + mbarriers / tile ids
};

// Tile iterator of the tile loop (executed by the producer thread only).
struct TileIter {
  int64_t cur = 0, end = 0, k = 0;
  bool started = false;
};

__device__ __forceinline__ int64_t next_tile(TileIter &it, const JacobiArgs &a, int64_t nt) {
  const int64_t p = gridDim.x, t = blockIdx.x;
  if (it.cur < it.end) return it.cur++;
  if (a.sched == SK_STATIC_BLOCK) {
    if (it.started) return -1;
    it.started = true;
    const int64_t q = nt / p, r = nt % p;
    it.cur = t * q + (t < r ? t : r);
    it.end = it.cur + q + (t < r ? 1 : 0);
  } else if (a.sched == SK_STATIC_CHUNK) {
    const int64_t kk = it.started ? it.k + p : t;
    it.started = true;
    it.k = kk;
    it.cur = kk * a.chunk;
    it.end = min(nt, it.cur + a.chunk);
  } else {
    const int64_t kk = (int64_t)atomicAdd(a.dyn_counter, 1ull);
    it.cur = kk * a.chunk;
    it.end = min(nt, it.cur + a.chunk);
  }
  if (it.cur >= it.end) return -1;
  return it.cur++;
}

// NST-deep producer / consumer ring of tile windows without CTA-wide
// barriers: the producer claims tiles in schedule order and loads tile m into
// slot m % NST once every unit warp has released the slot's previous tile
// (empty barrier); the unit warps wait only for their data (full barrier).  A
// tile id < 0 ends the loop (its full barrier completed by a plain arrive).
// PW: teams of up to 992 units get one extra warp whose lane 0 is the
// producer and executes no iterations (reading c34); larger teams produce
// from thread 0 between its own tiles, NST - 1 tiles ahead.
template <int BM, int BN, int NST, bool PW, bool TRACE>
__global__ void __launch_bounds__(1024) jacobi5_kernel(const __grid_constant__ JacobiArgs a,
                                                       const __grid_constant__ CUtensorMap tmc,
                                                       const __grid_constant__ CUtensorMap tmh) {
  using L = JLayout<BM, BN, NST>;
  extern __shared__ __align__(128) char smem[];
  uint64_t *bars = reinterpret_cast<uint64_t *>(smem + NST * L::BUF);   // full[NST], empty[NST]
  // per slot: tile id, first row / column of the tile, interior flag
  // (written by the producer before the slot's full barrier completes)
  volatile long long *tile_s = reinterpret_cast<volatile long long *>(smem + NST * L::BUF + 128);   // [NST][4]
  __shared__ unsigned s_last;
  const int64_t nt = a.ntr * a.ntc;
  const int units = a.units, u = threadIdx.x;
  const int cw = (units + 31) >> 5;          // warps holding units
  const int ptid = PW ? cw * 32 : 0;         // the producer thread
  TileIter it;

  auto issue = [&](int64_t i0, int64_t j0, int buf) {
    const int r0 = (int)(i0 - 1 - a.row0);   // local row of the box's first row
    const int c0 = (int)j0;
    char *b = smem + buf * L::BUF;
    tma_fence_proxy();
    tma_mbar_expect_tx(bars + buf, L::TX);
    tma_load_2d(b, &tmc, c0, r0, bars + buf);
    tma_load_2d(b + L::CEN, &tmh, c0 - 4, r0, bars + buf);
    tma_load_2d(b + L::CEN + L::HAL, &tmh, c0 + BN, r0, bars + buf);
  };

  // peer mode: sweeps this rank completed = sweeps each neighbour must have
  // delivered before a boundary tile may read / write halo rows
  unsigned long long gen = 0;
  auto peer_wait = [&](int64_t i0) {
    bool waited = false;
    if (a.win_up && a.halo_up_row >= i0 - 1 && a.halo_up_row <= i0 + BM) {
      wait_geq_sys(a.win + WIN_HALO_FROM_UP, gen);
      waited = true;
    }
    if (a.win_dn && a.halo_dn_row >= i0 - 1 && a.halo_dn_row <= i0 + BM) {
      wait_geq_sys(a.win + WIN_HALO_FROM_DN, gen);
      waited = true;
    }
    if (waited) fence_proxy_async_global();
  };
  int64_t prod = 0;   // producer: id of the tile it produced last
  auto produce = [&](int slot, bool wait_empty, unsigned parity) {
    const int64_t nx = next_tile(it, a, nt);
    if (wait_empty) {
      if (PW) tma_mbar_wait_backoff(bars + NST + slot, parity);
      else tma_mbar_wait(bars + NST + slot, parity);
    }
    tile_s[4 * slot] = nx;
    if (nx >= 0) {
      // interior tile: every position an iteration, no peer boundary row
      // tile id -> (row, column) of the tile grid: row-major (c24) or
      // column-major (UPIR_TILE_COLMAJOR, c35)
      // UPIR_TILE_REVERSE: id k enumerates the tiles from the last one (c36)
      const int64_t px = a.reverse ? nt - 1 - nx : nx;
      const int64_t i0 = (a.ti0 + (a.colmajor ? px % a.ntr : px / a.ntc)) * BM;
      const int64_t j0 = (a.tj0 + (a.colmajor ? px / a.ntr : px % a.ntc)) * BN;
      const bool fast = !TRACE && a.inner_chunk == 4 && (a.units & 31) == 0 && i0 >= a.lb0 && i0 + BM <= a.ub0 &&
                        j0 >= a.lb1 && j0 + BN <= a.ub1 && (a.ld & 3) == 0 && ((uintptr_t)a.out & 15) == 0 &&
                        (!a.win || ((a.send_up_row < i0 || a.send_up_row >= i0 + BM) &&
                                    (a.send_dn_row < i0 || a.send_dn_row >= i0 + BM)));
      tile_s[4 * slot + 1] = i0;
      tile_s[4 * slot + 2] = j0;
      tile_s[4 * slot + 3] = fast;
      if (a.win) peer_wait(i0);
      issue(i0, j0, slot);
    } else {
      tma_mbar_arrive(bars + slot);
    }
    prod = nx;
  };
  if (threadIdx.x == ptid) {
    if (a.win) gen = *reinterpret_cast<volatile unsigned long long *>(a.win + WIN_HALO_GEN);
    tma_prefetch_desc(&tmc);
    tma_prefetch_desc(&tmh);
#pragma unroll
    for (int b = 0; b < NST; ++b) {
      tma_mbar_init(bars + b, 1);
      // every thread of the unit warps releases the slot: the whole (rounded-up)
      // unit warps with a producer warp, all blockDim.x threads without one
      tma_mbar_init(bars + NST + b, PW ? cw * 32 : blockDim.x);
    }
    tma_fence_init();
  }
  __syncthreads();

  const int ic = a.inner_chunk;
  constexpr int POS = BM * BN;
  if (PW && threadIdx.x >= cw * 32) {
    if (threadIdx.x == ptid)
      for (int64_t m = 0; prod >= 0; ++m) {
        const int slot = (int)(m % NST);
        produce(slot, m >= NST, (unsigned)(((m - NST) / NST) & 1));
      }
  } else {
    if (!PW && threadIdx.x == 0)
      for (int k = 0; k < NST - 1 && prod >= 0; ++k) produce(k, false, 0);
    for (int iter = 0;; ++iter) {
      const int buf = iter % NST;
      if (!PW && threadIdx.x == 0 && prod >= 0) {
        // tile of iteration iter + NST - 1 into the slot iteration iter - 1 used
        const int slot = (iter + NST - 1) % NST;
        produce(slot, iter >= 1, (unsigned)(((iter - 1) / NST) & 1));
      }
      tma_mbar_wait(bars + buf, (unsigned)((iter / NST) & 1));
      const int64_t tile = tile_s[4 * buf];
      if (tile < 0) break;
      const int64_t i0 = tile_s[4 * buf + 1], j0 = tile_s[4 * buf + 2];
      const bool fast = tile_s[4 * buf + 3] != 0;
      const float *cen = reinterpret_cast<const float *>(smem + buf * L::BUF);
      const float *lef = reinterpret_cast<const float *>(smem + buf * L::BUF + L::CEN);
      const float *rig = reinterpret_cast<const float *>(smem + buf * L::BUF + L::CEN + L::HAL);
      auto at = [&](int r, int c) -> float {   // smem row r (global row i0-1+r), tile column c in [-1, BN]
        if (c < 0) return lef[r * 4 + 3];
        if (c >= BN) return rig[r * 4 + (c - BN)];
        return cen[r * BN + c];
      };
      // interior tile: static,4 chunks with tile-relative int32 indexing; the
      // west / east neighbours come from the adjacent lanes' vectors (warp
      // shuffles), from shared memory only at the warp's edge lanes or the
      // halo columns
      if (fast) {
        float *obase = a.out + (i0 - a.row0) * a.ld + j0;
        const int ld = (int)a.ld;
        const int lane = threadIdx.x & 31;
#pragma unroll 4
        for (int k = u; k * 4 < POS; k += units) {
          const int r = (k * 4) / BN, c = (k * 4) % BN;
          const float *pc = cen + r * BN + c;
          const float4 up = *reinterpret_cast<const float4 *>(pc);
          const float4 md = *reinterpret_cast<const float4 *>(pc + BN);
          const float4 dn = *reinterpret_cast<const float4 *>(pc + 2 * BN);
          float w0 = __shfl_up_sync(0xffffffffu, md.w, 1);
          float e3 = __shfl_down_sync(0xffffffffu, md.x, 1);
          if (c == 0) w0 = lef[(r + 1) * 4 + 3];
          else if (lane == 0) w0 = pc[BN - 1];
          if (c + 4 == BN) e3 = rig[(r + 1) * 4];
          else if (lane == 31) e3 = pc[BN + 4];
          float4 o;
          o.x = __fmul_rn(0.25f, __fadd_rn(__fadd_rn(up.x, dn.x), __fadd_rn(w0, md.y)));
          o.y = __fmul_rn(0.25f, __fadd_rn(__fadd_rn(up.y, dn.y), __fadd_rn(md.x, md.z)));
          o.z = __fmul_rn(0.25f, __fadd_rn(__fadd_rn(up.z, dn.z), __fadd_rn(md.y, md.w)));
          o.w = __fmul_rn(0.25f, __fadd_rn(__fadd_rn(up.w, dn.w), __fadd_rn(md.z, e3)));
          __stcs(reinterpret_cast<float4 *>(obase + (int64_t)r * ld + c), o);
        }
      } else if (ic == 4) {
        // static,4 over units: chunk k = 4 consecutive columns of one row
        for (int k = u; u < units && k * 4 < POS; k += units) {
          const int r = (k * 4) / BN, c = (k * 4) % BN;
          const int64_t i = i0 + r;
          if (i < a.lb0 || i >= a.ub0) continue;
          const int64_t j = j0 + c;
          if (j + 3 < a.lb1 || j >= a.ub1) continue;
          const float4 up = *reinterpret_cast<const float4 *>(cen + r * BN + c);
          const float4 dn = *reinterpret_cast<const float4 *>(cen + (r + 2) * BN + c);
          const float4 md = *reinterpret_cast<const float4 *>(cen + (r + 1) * BN + c);
          const float w0 = at(r + 1, c - 1), e3 = at(r + 1, c + 4);
          float4 o;
          o.x = __fmul_rn(0.25f, __fadd_rn(__fadd_rn(up.x, dn.x), __fadd_rn(w0, md.y)));
          o.y = __fmul_rn(0.25f, __fadd_rn(__fadd_rn(up.y, dn.y), __fadd_rn(md.x, md.z)));
          o.z = __fmul_rn(0.25f, __fadd_rn(__fadd_rn(up.z, dn.z), __fadd_rn(md.y, md.w)));
          o.w = __fmul_rn(0.25f, __fadd_rn(__fadd_rn(up.w, dn.w), __fadd_rn(md.z, e3)));
          float *dst = a.out + (i - a.row0) * a.ld + j;
          // peer mode: my boundary rows also land in the neighbour's halo row
          float *pdst = (a.win && i == a.send_up_row && a.peer_up) ? a.peer_up + (i - a.peer_up_row0) * a.ld + j
                                                                    : nullptr;
          float *pdst2 = (a.win && i == a.send_dn_row && a.peer_dn) ? a.peer_dn + (i - a.peer_dn_row0) * a.ld + j
                                                                     : nullptr;
          if (j >= a.lb1 && j + 4 <= a.ub1) {
            __stcs(reinterpret_cast<float4 *>(dst), o);
            if (pdst) *reinterpret_cast<float4 *>(pdst) = o;
            if (pdst2) *reinterpret_cast<float4 *>(pdst2) = o;
          } else {
            const float ov[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (j + q >= a.lb1 && j + q < a.ub1) {
                dst[q] = ov[q];
                if (pdst) pdst[q] = ov[q];
                if (pdst2) pdst2[q] = ov[q];
              }
          }
          if constexpr (TRACE) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              if (j + q >= a.lb1 && j + q < a.ub1) {
                const int64_t idx = tile * POS + r * BN + c + q;
                a.trace[idx] = blockIdx.x;
                a.trace[nt * POS + idx] = u;
                atomicAdd(a.trace + 2 * nt * POS + idx, 1);
              }
          }
        }
      } else {
        // static,ic over units, element by element
        for (int64_t k = u; u < units && k * ic < POS; k += units) {
          for (int pos = (int)(k * ic); pos < (int)min((int64_t)POS, (k + 1) * ic); ++pos) {
            const int r = pos / BN, c = pos % BN;
            const int64_t i = i0 + r, j = j0 + c;
            if (i < a.lb0 || i >= a.ub0 || j < a.lb1 || j >= a.ub1) continue;
            const float v = __fmul_rn(0.25f, __fadd_rn(__fadd_rn(at(r, c), at(r + 2, c)),
                                                       __fadd_rn(at(r + 1, c - 1), at(r + 1, c + 1))));
            a.out[(i - a.row0) * a.ld + j] = v;
            if (a.win) {
              if (i == a.send_up_row && a.peer_up) a.peer_up[(i - a.peer_up_row0) * a.ld + j] = v;
              if (i == a.send_dn_row && a.peer_dn) a.peer_dn[(i - a.peer_dn_row0) * a.ld + j] = v;
            }
            if constexpr (TRACE) {
              const int64_t idx = tile * POS + pos;
              a.trace[idx] = blockIdx.x;
              a.trace[nt * POS + idx] = u;
              atomicAdd(a.trace + 2 * nt * POS + idx, 1);
            }
          }
        }
      }
      // this thread is done with `buf` (its window reads and its read of the
      // slot record): a per-thread release, so the producer's refill is
      // ordered after every read without relying on a warp barrier
      tma_mbar_arrive(bars + NST + buf);
    }
  }
  // peer mode: after the whole sweep (every unit's peer stores fenced), the
  // last team counts the sweep and delivers it to both neighbours
  if (a.win) {
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned long long t = atomicAdd(a.win + WIN_HALO_DONE, 1ull);
      if (t == (unsigned long long)gridDim.x - 1) {
        a.win[WIN_HALO_DONE] = 0ull;
        __threadfence_system();
        const unsigned long long g = *reinterpret_cast<volatile unsigned long long *>(a.win + WIN_HALO_GEN);
        *reinterpret_cast<volatile unsigned long long *>(a.win + WIN_HALO_GEN) = g + 1ull;
        if (a.win_up) red_release_sys_add(a.win_up + WIN_HALO_FROM_DN, 1ull);
        if (a.win_dn) red_release_sys_add(a.win_dn + WIN_HALO_FROM_UP, 1ull);
      }
    }
  }
  // dynamic: the last team resets the tile counter for the next launch
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

template <int BM, int BN, int NST>
cudaError_t launch_nst(const JacobiArgs &a, const CUtensorMap &c, const CUtensorMap &h, int teams, int units,
                       bool trace, cudaStream_t s) {
  using L = JLayout<BM, BN, NST>;
  const bool pw = units <= 992;
  auto k = pw ? jacobi5_kernel<BM, BN, NST, true, false> : jacobi5_kernel<BM, BN, NST, false, false>;
  if constexpr (NST == 2) {   // traced runs (tests) use the 2-deep ring
    if (trace) k = pw ? jacobi5_kernel<BM, BN, NST, true, true> : jacobi5_kernel<BM, BN, NST, false, true>;
  }
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
  if (e != cudaSuccess) return e;
  JacobiArgs b = a;
  b.units = units;
  const int threads = pw ? (units + 31) / 32 * 32 + 32 : units;   // + the producer warp
  k<<<teams, threads, L::SMEM, s>>>(b, c, h);
  return cudaGetLastError();
}

// Ring depth: the deepest ring that keeps at most ~112 KB of tile windows per
// SM (teams resident per SM x NST x window bytes).  Measured on B200 (C3,
// tools/experiments/jacobi_sweep.py): 3 teams/SM x 2 slots and 2 teams/SM x 3 slots
// of 16x256 tiles are best; deeper rings at the same residency lose 10-15 %
// (more reads queued ahead of the write-back stream).
template <int BM, int BN>
cudaError_t launch_bmbn(const JacobiArgs &a, const CUtensorMap &c, const CUtensorMap &h, int teams, int units,
                        bool trace, cudaStream_t s) {
  int nst = 0;
  if (const char *v = getenv("UPIR_JACOBI_NST")) nst = atoi(v);
  if (trace) {
    nst = 2;
  } else if (nst < 2 || nst > 4) {
    const int per_sm = teams >= 148 ? (teams + 147) / 148 : 1;   // teams resident per SM (148 SMs)
    const int smem_budget = 227 * 1024 / per_sm - 1024;
    nst = 2;
    for (int d = 4; d > 2; --d) {
      const int sm = d == 4 ? JLayout<BM, BN, 4>::SMEM : JLayout<BM, BN, 3>::SMEM;
      if (sm <= smem_budget && per_sm * d * JLayout<BM, BN, 2>::TX <= 112 * 1024) {
        nst = d;
        break;
      }
    }
  }
  if (nst == 4) return launch_nst<BM, BN, 4>(a, c, h, teams, units, trace, s);
  if (nst == 3) return launch_nst<BM, BN, 3>(a, c, h, teams, units, trace, s);
  return launch_nst<BM, BN, 2>(a, c, h, teams, units, trace, s);
}

}  // namespace

bool jacobi_supported_tile(int bm, int bn) {
  return (bm == 32 && bn == 256) || (bm == 32 && bn == 128) || (bm == 16 && bn == 256) || (bm == 64 && bn == 128) ||
         (bm == 8 && bn == 64);
}

cudaError_t launch_jacobi_tma(const JacobiArgs &a, const void *tmc, const void *tmh, int teams, int units, int bm,
                              int bn, bool trace, cudaStream_t s) {
  const CUtensorMap &c = *reinterpret_cast<const CUtensorMap *>(tmc);
  const CUtensorMap &h = *reinterpret_cast<const CUtensorMap *>(tmh);
  if (bm == 32 && bn == 256) return launch_bmbn<32, 256>(a, c, h, teams, units, trace, s);
  if (bm == 32 && bn == 128) return launch_bmbn<32, 128>(a, c, h, teams, units, trace, s);
  if (bm == 16 && bn == 256) return launch_bmbn<16, 256>(a, c, h, teams, units, trace, s);
  if (bm == 64 && bn == 128) return launch_bmbn<64, 128>(a, c, h, teams, units, trace, s);
  if (bm == 8 && bn == 64) return launch_bmbn<8, 64>(a, c, h, teams, units, trace, s);
  return cudaErrorInvalidValue;
}

}  // namespace upir
