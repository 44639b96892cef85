// k_stencil.cu -- the STENCIL2D loop body (the paper's
// "2D stencil, filter size = 7"; reading c28):
//   out[i][j] = sum_{a,b in [-R,R]} w[a+R][b+R] * in[i+a][j+b]
// over a tiled collapse(2) upir.loop (reading c24: tiles anchored at 0, tile
// loop over TEAMS, box positions static,ic over UNITS).  Each team stages the
// (BM+2R) x (BN+8) input window of its tile in shared memory with one TMA
// tensor load (zero fill out of range), double-buffered: one elected thread
// has the next tile's window in flight while the team computes the current
// one; the F x F weights are staged once; each unit produces 4 consecutive
// outputs per chunk from registers
// (register-blocked taps, fp32 FMA in the fixed order of the filter rows /
// columns).  49 FMAs per point at F = 7: ALU-bound rather than HBM-bound.
#include "dev_tma.cuh"
#include "upir_internal.h"

namespace upir {
namespace {

template <int R, int BM, int BN>
struct SLayout {
  static constexpr int F = 2 * R + 1, WR = BM + 2 * R, WC = BN + 8;
  // TMA boxes are at most 256 columns wide: a wide window is NB boxes of 256
  // columns plus one of 8, each landing as its own dense [WR][box] block
  static constexpr bool WIDE = WC > 256;
  static constexpr int NB = WIDE ? (WC - 8) / 256 : 0;
  // strip layout (BN = 4 * units): one dense [WR][SW] block per warp holding
  // the warp's 128 output columns plus 4 halo columns each side
  static constexpr int SW = 136, NS = BN / 128;
  static constexpr int SBLK = (WR * SW * 4 + 127) / 128 * 128;   // TMA destinations are 128-B aligned
  static constexpr int STX = WR * SW * 4 * (NS > 0 ? NS : 1);    // bytes one strip window delivers
  static constexpr int GBUF = WR * WC * 4, SBUF = SBLK * (NS > 0 ? NS : 1);
  static constexpr int BUF = (((GBUF > SBUF ? GBUF : SBUF)) + 127) / 128 * 128;
  // pipeline depth (window buffers)
  static constexpr int NST = 2;   // 3 stages measured slower (they cost resident CTAs per SM)
  static constexpr int SMEM = NST * BUF + 256 + F * F * 4 + 128;
};

// smem offset (floats) of window (row, col) -- col a multiple of 4 for vectors
template <int R, int BM, int BN>
__device__ __forceinline__ int win_off(int row, int col) {
  using L = SLayout<R, BM, BN>;
  if constexpr (!L::WIDE) {
    return row * L::WC + col;
  } else {
    const int sub = col >> 8;
    if (sub < L::NB) return sub * (L::WR * 256) + row * 256 + (col & 255);
    return L::NB * (L::WR * 256) + row * 8 + (col - L::NB * 256);
  }
}

// MAXT: the team size the kernel is compiled for (256 lets the 49 taps stay
// in registers; 1024 caps registers at 64 for teams of up to 1024 units).
// PW: teams of up to 256 units get one extra warp whose lane 0 is a
// dedicated TMA producer (it executes no iterations); larger teams produce
// from thread 0 between its own tiles.
template <int R, int BM, int BN, int MAXT, bool PW = (MAXT <= 256)>
__global__ void __launch_bounds__(MAXT + (PW ? 32 : 0)) stencil_kernel(const __grid_constant__ StencilArgs a,
                                                       const __grid_constant__ CUtensorMap tmw,
                                                       const __grid_constant__ CUtensorMap tmw8,
                                                       const __grid_constant__ CUtensorMap tms) {
  // window column c holds global column j0 - 4 + c (4-aligned so that a
  // unit's taps are read as 16-B vectors)
  using L = SLayout<R, BM, BN>;
  constexpr int F = L::F, WR = L::WR, WCP = L::WC;
  extern __shared__ __align__(128) char smc[];
  constexpr int NST = L::NST;
  // full[NST][NWB] (TMA landed / end marker; strip path: one barrier per warp
  // strip, so a warp waits only for its own box), empty[NST] (every unit-warp
  // thread done with the buffer)
  constexpr int NWB = L::NS > 0 ? L::NS : 1;
  uint64_t *full = reinterpret_cast<uint64_t *>(smc + NST * L::BUF);
  uint64_t *empty = full + NST * NWB;
  static_assert((NST * NWB + NST) * 8 <= 192, "barrier block");
  // per slot: tile id, first row, first column (written by the producer
  // before the slot's full barriers complete)
  volatile long long *tile_s = reinterpret_cast<volatile long long *>(smc + NST * L::BUF + 192);   // [NST][3]
  float *w = reinterpret_cast<float *>(smc + NST * L::BUF + 256);
  __shared__ unsigned s_last;
  const int units = a.units, u = threadIdx.x;
  const int cw = (units + 31) >> 5;            // warps holding units
  const int ptid = PW ? cw * 32 : 0;           // the producer thread
  for (int e = threadIdx.x; e < F * F; e += blockDim.x) w[e] = a.w[e];
  __syncthreads();
  float wr[F * F];   // the taps live in registers for the whole kernel
#pragma unroll
  for (int e = 0; e < F * F; ++e) wr[e] = w[e];
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
  // strip path: static,4 with BN = 4 * units -- unit u owns columns 4u..4u+3
  // (traced runs take the generic static,4 path: same position -> unit map)
  const bool strip = a.inner_chunk == 4 && BN == 4 * units && BN % 128 == 0 && MAXT <= 256 && !a.trace;
  auto issue = [&](int64_t i0, int64_t j0, int buf) {
    tma_fence_proxy();
    if (strip) {
#pragma unroll 1
      for (int w = 0; w < L::NS; ++w) {
        tma_mbar_expect_tx(full + buf * NWB + w, L::STX / L::NS);
        tma_load_2d(smc + buf * L::BUF + w * L::SBLK, &tms, (int)(j0 - 4 + 128 * w), (int)(i0 - R - a.row0),
                    full + buf * NWB + w);
      }
      return;
    }
    uint64_t *bar0 = full + buf * NWB;
    tma_mbar_expect_tx(bar0, WR * WCP * 4);
    // window rows [i0-R, i0+BM+R) x cols [j0-4, j0+BN+4) of the local buffer
    if constexpr (!L::WIDE) {
      tma_load_2d(smc + buf * L::BUF, &tmw, (int)(j0 - 4), (int)(i0 - R - a.row0), bar0);
    } else {
#pragma unroll
      for (int q = 0; q < L::NB; ++q)
        tma_load_2d(smc + buf * L::BUF + q * (WR * 256 * 4), &tmw, (int)(j0 - 4 + 256 * q), (int)(i0 - R - a.row0),
                    bar0);
      tma_load_2d(smc + buf * L::BUF + L::NB * (WR * 256 * 4), &tmw8, (int)(j0 - 4 + 256 * L::NB),
                  (int)(i0 - R - a.row0), bar0);
    }
  };
  if (threadIdx.x == ptid) {
    tma_prefetch_desc(&tmw);
    if constexpr (L::WIDE) tma_prefetch_desc(&tmw8);
    if (strip) tma_prefetch_desc(&tms);
#pragma unroll
    for (int b = 0; b < NST; ++b) {
#pragma unroll
      for (int w = 0; w < NWB; ++w) tma_mbar_init(full + b * NWB + w, 1);
      // every thread of the unit warps releases the slot: the whole (rounded-up)
      // unit warps with a producer warp, all blockDim.x threads without one
      tma_mbar_init(empty + b, PW ? cw * 32 : blockDim.x);
    }
    tma_fence_init();
  }
  __syncthreads();
  // Producer / consumer ring of NST window buffers without CTA-wide
  // barriers: thread 0 claims tiles NST - 1 ahead and loads each into the
  // buffer every warp has released (empty barrier); the warps wait only for
  // their data (full barrier).  A tile id < 0 ends the loop (its full
  // barrier completed by a plain arrive).
  int64_t prod = 0;   // thread 0: id of the tile it produced last
  auto produce = [&](int slot, bool wait_empty, unsigned parity) {
    const int64_t nx = next_tile();
    if (wait_empty) {
      if (PW) tma_mbar_wait_backoff(empty + slot, parity);
      else tma_mbar_wait(empty + slot, parity);
    }
    tile_s[3 * slot] = nx;
    if (nx >= 0) {
      // the tile's origin, computed once here (the unit warps read it)
      const int64_t i0 = (a.ti0 + nx / a.ntc) * BM, j0 = (a.tj0 + nx % a.ntc) * BN;
      tile_s[3 * slot + 1] = i0;
      tile_s[3 * slot + 2] = j0;
      issue(i0, j0, slot);
    } else {
#pragma unroll
      for (int w = 0; w < NWB; ++w) tma_mbar_arrive(full + slot * NWB + w);
    }
    prod = nx;
  };
  if (PW && threadIdx.x >= cw * 32) {
    // dedicated producer: tile m into slot m % NST once every unit warp has
    // released that slot's previous tile (m - NST)
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
      // tile of iteration iter + NST - 1 into the buffer iteration iter - 1 used
      const int slot = (iter + NST - 1) % NST;
      produce(slot, iter >= 1, (unsigned)(((iter - 1) / NST) & 1));
    }
    tma_mbar_wait(full + buf * NWB + (strip ? (u >> 5) % NWB : 0), (unsigned)((iter / NST) & 1));
    const int64_t tile = tile_s[3 * buf];
    if (tile < 0) break;
    const float *win = reinterpret_cast<const float *>(smc + buf * L::BUF);
    const int64_t i0 = tile_s[3 * buf + 1], j0 = tile_s[3 * buf + 2];
    const int ic = a.inner_chunk;
    if (strip) {
      // static,4 with BN = 4 * units: unit u owns the 4-column strip c = 4u of
      // every tile row (chunk k = r*units + u), visited top to bottom in
      // blocks of H output rows.  The H + F - 1 input rows of a block stream
      // through registers once (3 LDS.128 each) and each feeds the output
      // rows it touches: H x 4 independent accumulator chains in flight, and
      // the unrolled block body (H * F * F * 4 FFMA, weights in uniform
      // registers) stays inside the 32 KB L1.5 instruction cache -- a fully
      // unrolled tile does not (measured: 'no instruction' stalls).
      // Per output the taps accumulate in the order filter row 0..F-1,
      // column 0..F-1 from 0 -- the same sequence as the other paths.
      constexpr int H = 4;   // H = 8 measured slower (code size, registers)
      static_assert(BM % H == 0, "tile height must be a multiple of the row block");
      const int c = 4 * u;
      const int64_t j = j0 + c;
      const bool jok = j + 3 >= a.lb1 && j < a.ub1;
      // this unit's columns in its warp's strip block: compile-time offsets per (row, vector)
      const float *sbase = win + (u >> 5) * (L::SBLK / 4) + (u & 31) * 4;
      // a tile inside the iteration space with aligned rows stores without checks
      const int64_t ld = a.ld;
      float *dst0 = a.out + (i0 - a.row0) * ld + j;
      const bool interior = i0 >= a.lb0 && i0 + BM <= a.ub0 && j0 >= a.lb1 && j0 + BN <= a.ub1 && (ld & 3) == 0 &&
                            ((uintptr_t)a.out & 15) == 0;
#pragma unroll 1
      for (int r0 = 0; r0 < BM; r0 += H) {
        float acc[H][4];
#pragma unroll
        for (int h = 0; h < H; ++h)
#pragma unroll
          for (int t = 0; t < 4; ++t) acc[h][t] = 0.f;
#pragma unroll
        for (int p = 0; p < H + F - 1; ++p) {   // window row r0 + p
          float v[12];
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const float4 t4 = *reinterpret_cast<const float4 *>(sbase + (r0 + p) * L::SW + 4 * q);
            v[4 * q] = t4.x;
            v[4 * q + 1] = t4.y;
            v[4 * q + 2] = t4.z;
            v[4 * q + 3] = t4.w;
          }
          // q outermost: the H x 4 chains of this input row interleave (each
          // output still takes its taps in (filter row, column) order)
#pragma unroll
          for (int q = 0; q < F; ++q)
#pragma unroll
            for (int h = 0; h < H; ++h) {
              const int pp = p - h;   // filter row feeding block row h
              if (pp >= 0 && pp < F) {
#pragma unroll
                for (int t = 0; t < 4; ++t) acc[h][t] = __fmaf_rn(wr[pp * F + q], v[4 - R + t + q], acc[h][t]);
              }
            }
        }
        float *dstb = dst0 + r0 * ld;
        if (interior) {
#pragma unroll
          for (int h = 0; h < H; ++h)
            __stcs(reinterpret_cast<float4 *>(dstb + h * ld), make_float4(acc[h][0], acc[h][1], acc[h][2], acc[h][3]));
        } else {
#pragma unroll
          for (int h = 0; h < H; ++h) {
            const int64_t i = i0 + r0 + h;
            if (jok && i >= a.lb0 && i < a.ub0) {
              float *dst = dstb + h * ld;
              if (j >= a.lb1 && j + 4 <= a.ub1 && ((uintptr_t)dst & 15) == 0) {
                __stcs(reinterpret_cast<float4 *>(dst), make_float4(acc[h][0], acc[h][1], acc[h][2], acc[h][3]));
              } else {
#pragma unroll
                for (int t = 0; t < 4; ++t)
                  if (j + t >= a.lb1 && j + t < a.ub1) dst[t] = acc[h][t];
              }
            }
          }
        }
      }
    } else if (ic == 4) {
      for (int k = u; u < units && k * 4 < POS; k += units) {
        const int r = (k * 4) / BN, c = (k * 4) % BN;
        const int64_t i = i0 + r, j = j0 + c;
        if (i < a.lb0 || i >= a.ub0 || j + 3 < a.lb1 || j >= a.ub1) continue;
        float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int p = 0; p < F; ++p) {
          // window columns c .. c+11 = global j-4 .. j+7 as three 16-B vectors
          float v[12];
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            const float4 t4 = *reinterpret_cast<const float4 *>(win + win_off<R, BM, BN>(r + p, c + 4 * q));
            v[4 * q] = t4.x;
            v[4 * q + 1] = t4.y;
            v[4 * q + 2] = t4.z;
            v[4 * q + 3] = t4.w;
          }
#pragma unroll
          for (int q = 0; q < F; ++q) {
            const float wq = wr[p * F + q];
#pragma unroll
            for (int t = 0; t < 4; ++t) acc[t] = __fmaf_rn(wq, v[4 - R + t + q], acc[t]);
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
      for (int64_t k = u; u < units && k * ic < POS; k += units) {
        for (int pos = (int)(k * ic); pos < (int)min((int64_t)POS, (k + 1) * ic); ++pos) {
          const int r = pos / BN, c = pos % BN;
          const int64_t i = i0 + r, j = j0 + c;
          if (i < a.lb0 || i >= a.ub0 || j < a.lb1 || j >= a.ub1) continue;
          float acc = 0.f;
          for (int p = 0; p < F; ++p)
            for (int q = 0; q < F; ++q) acc = __fmaf_rn(w[p * F + q], win[win_off<R, BM, BN>(r + p, c + 4 - R + q)], acc);
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
    tma_mbar_arrive(empty + buf);   // this thread is done with `buf` (per-thread release)
  }
  }   // unit warps
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
  using L = SLayout<R, BM, BN>;
  CUtensorMap tm, tm8, tms;
  if (!encode_tmap_2d(&tms, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, a.in, (uint64_t)a.nx, (uint64_t)(a.ny - a.row0),
                      (uint64_t)a.ld * 4, L::SW, L::WR, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B))
    return cudaErrorInvalidValue;
  if (!encode_tmap_2d(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, a.in, (uint64_t)a.nx, (uint64_t)(a.ny - a.row0),
                      (uint64_t)a.ld * 4, L::WIDE ? 256 : L::WC, L::WR, CU_TENSOR_MAP_SWIZZLE_NONE,
                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B) ||
      !encode_tmap_2d(&tm8, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, a.in, (uint64_t)a.nx, (uint64_t)(a.ny - a.row0),
                      (uint64_t)a.ld * 4, 8, L::WR, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B))
    return cudaErrorInvalidValue;
  auto k = (BN == 512 && units == 128)   ? stencil_kernel<R, BM, BN, 128>
           : units <= 256                 ? stencil_kernel<R, BM, BN, 256>
                                          : stencil_kernel<R, BM, BN, 1024>;
  const int threads = units <= 256 ? (units + 31) / 32 * 32 + 32 : units;   // + the producer warp
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
  if (e != cudaSuccess) return e;
  StencilArgs b = a;
  b.units = units;
  k<<<teams, threads, L::SMEM, s>>>(b, tm, tm8, tms);
  return cudaGetLastError();
}

}  // namespace

bool stencil_supported(int F, int bm, int bn) {
  return (F == 3 || F == 5 || F == 7) &&
         ((bm == 16 && bn == 128) || (bm == 8 && bn == 64) || (bm == 16 && bn == 512) || (bm == 16 && bn == 1024) ||
          (bm == 8 && bn == 512) || (bm == 8 && bn == 1024) || (bm == 8 && bn == 256) || (bm == 4 && bn == 512) ||
          (bm == 4 && bn == 256));
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
  UPIR_ST(1, 16, 512)
  UPIR_ST(2, 16, 512)
  UPIR_ST(3, 16, 512)
  UPIR_ST(1, 16, 1024)
  UPIR_ST(2, 16, 1024)
  UPIR_ST(3, 16, 1024)
  UPIR_ST(1, 8, 512)
  UPIR_ST(2, 8, 512)
  UPIR_ST(3, 8, 512)
  UPIR_ST(1, 8, 1024)
  UPIR_ST(2, 8, 1024)
  UPIR_ST(3, 8, 1024)
  UPIR_ST(1, 8, 256)
  UPIR_ST(2, 8, 256)
  UPIR_ST(3, 8, 256)
  UPIR_ST(1, 4, 512)
  UPIR_ST(2, 4, 512)
  UPIR_ST(3, 4, 512)
  UPIR_ST(1, 4, 256)
  UPIR_ST(2, 4, 256)
  UPIR_ST(3, 4, 256)
#undef UPIR_ST
  return cudaErrorInvalidValue;
}

}  // namespace upir
