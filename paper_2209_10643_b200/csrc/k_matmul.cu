// k_matmul.cu -- the MATMUL loop body on the 5th-generation tensor cores:
//   C[i][j] = sum_k A[i][k] * B[k][j]      (north_star; c17)
// as a collapse(2) upir.loop over (i, j) whose tile loop (128 x 256 output
// tiles anchored at 0) is scheduled over persistent TEAMS (CTAs); inside a
// tile the work is cooperative (reading c24).
//
// sm_100a design (one CTA per SM, 256 threads for bf16, 384 for fp32):
//   warp 0      : TMA producer -- A tile 128 x 64 (K-major) and B tile 64 x 256
//                 (N-major, four 64-column boxes), 128-B swizzle, 4-stage
//                 mbarrier ring (full / empty).
//   warp 1      : one elected thread issues tcgen05.mma.cta_group::1.kind::f16
//                 (M=128, N=256, K=16) from shared-memory descriptors into a
//                 TMEM accumulator; tcgen05.commit frees smem stages and
//                 signals the epilogue.  Two accumulators (2 x 256 columns)
//                 so the epilogue of tile t overlaps the MMAs of tile t+1.
//   warp 2      : TMEM allocator (512 columns).
//   warps 4..7  : epilogue -- tcgen05.ld 32x32b.x32 (TMEM lane = output row)
//                 -> registers -> fp32 C with 256-bit stores (masked at ragged
//                 edges).
// bf16 inputs, fp32 accumulation (kind::f16); fp32 inputs via 3xTF32
// (kind::tf32) over operands pre-split into tf32 hi / lo copies by
// tf32_split_kernel (warps 8..11 of the 384-unit team have no role).
// Ragged M/N/K are handled by TMA zero fill (loads) and masks (stores).
#include "dev_tma.cuh"
#include "upir_internal.h"

namespace upir {
namespace {

// Per-dtype configuration.  BF16: kind::f16, K = 16 per MMA, 64-deep stages.
// F32 (3xTF32): kind::tf32, K = 8 per MMA, 32-deep stages; each stage holds
// the hi = rna_tf32(x) and lo = x - hi copies of the operand tiles (split
// once in HBM by tf32_split_kernel), and D += lo_a*hi_b + hi_a*lo_b +
// hi_a*hi_b (small terms first), which keeps the fp32 result within the
// 1e-5 bar.
template <int DT>
struct Cfg;
template <>
struct Cfg<UPIR_BF16> {
  static constexpr int ES = 2, BK = 64, STAGES = 4, THREADS = 256, KSTEP = 16;
  static constexpr int NSPLIT = 1;   // operand copies per stage (hi only)
  static constexpr uint32_t FMT = 1;  // BF16
};
template <>
struct Cfg<UPIR_F32> {
  static constexpr int ES = 4, BK = 32, STAGES = 2, THREADS = 384, KSTEP = 8;
  static constexpr int NSPLIT = 2;   // hi and lo copies
  static constexpr uint32_t FMT = 2;  // TF32
};

constexpr int BM = 128, BN = 256;
constexpr uint32_t TMEM_COLS = 512;

template <int DT>
struct MLayout {
  using C = Cfg<DT>;
  static constexpr int A_BYTES = BM * C::BK * C::ES;              // one copy of the A tile
  static constexpr int BOXN = 128 / C::ES;                        // N columns per 128-B swizzle atom
  static constexpr int B_BOX = BOXN * C::BK * C::ES;              // one B box (BOXN x BK)
  static constexpr int B_BYTES = C::BK * BN * C::ES;            // B tile (BN / BOXN boxes)
  static constexpr int COPY = A_BYTES + B_BYTES;                  // A + B of one split copy
  static constexpr int STAGE = COPY * C::NSPLIT;
  static constexpr int SMEM = C::STAGES * STAGE + 1024 + 256;
  static constexpr int TX = COPY * C::NSPLIT;                     // bytes TMA delivers per stage
};

// UMMA shared-memory layout types (descriptor bits [61,64))
constexpr uint64_t LT_SW128 = 2, LT_SW128_BASE32B = 1;

__device__ __forceinline__ uint64_t smem_desc(const void *p, uint32_t lbo, uint32_t sbo, uint64_t lt = LT_SW128) {
  // tcgen05 shared-memory matrix descriptor: start >> 4 [0,14), LBO >> 4
  // [16,30), SBO >> 4 [32,46), version 1 [46,48), base offset 0, layout
  // type at [61,64).
  const uint64_t a = (uint64_t)((tma_smem(p) >> 4) & 0x3FFF);
  return a | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) | ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) |
         (lt << 61);
}

// instruction descriptor: D f32, A/B fmt, A K-major, B MN-major, N=256, M=128
template <int DT>
constexpr uint32_t idesc() {
  return (1u << 4) | (Cfg<DT>::FMT << 7) | (Cfg<DT>::FMT << 10) | (0u << 15) | (1u << 16) |
         ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
}

template <int DT>
__device__ __forceinline__ void mma(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  if constexpr (DT == UPIR_BF16)
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc<DT>()), "r"(accum));
  else
    asm volatile(
        "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
        " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc<DT>()), "r"(accum));
}
// round-to-nearest (ties away) to tf32, returned as an fp32 bit pattern
__device__ __forceinline__ float to_tf32(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

__device__ __forceinline__ void mma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(tma_smem(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
}

// Tile id -> (tile row, tile column) (reading c32): ids enumerate the tiles
// in groups of GROUP tile rows, column-major inside a group -- a tiling of
// the tile loop that keeps the tiles running at the same
// time on a ~GROUP x 10 block, whose A rows and B columns fit in L2.
constexpr int64_t GROUP = 16;
__device__ __forceinline__ void tile_coords(int64_t tile, int64_t ntr, int64_t ntc, int64_t &ti, int64_t &tj) {
  const int64_t per = GROUP * ntc;
  const int64_t g = tile / per, w = tile % per;
  const int64_t rows = min(GROUP, ntr - g * GROUP);   // last group may be short
  ti = g * GROUP + w % rows;
  tj = w / rows;
}

// Tile sequence of this team under a static tile schedule (reading c24).
struct TileSeq {
  int64_t cur, end, k;
  int sched;
  int64_t chunk, nt, p, t;
  __device__ void init(int sched_, int64_t chunk_, int64_t nt_) {
    sched = sched_;
    chunk = chunk_;
    nt = nt_;
    p = gridDim.x;
    t = blockIdx.x;
    if (sched == SK_STATIC_BLOCK) {
      const int64_t q = nt / p, r = nt % p;
      cur = t * q + (t < r ? t : r);
      end = cur + q + (t < r ? 1 : 0);
      k = 0;
    } else {
      k = t;
      cur = k * chunk;
      end = min(nt, cur + chunk);
    }
  }
  __device__ int64_t next() {
    while (true) {
      if (cur < end) return cur++;
      if (sched == SK_STATIC_BLOCK) return -1;
      k += p;
      cur = k * chunk;
      if (cur >= nt) return -1;
      end = min(nt, cur + chunk);
    }
  }
};

template <int DT>
__global__ void __launch_bounds__(Cfg<DT>::THREADS, 1)
    matmul_kernel(const __grid_constant__ MatmulArgs a, const __grid_constant__ CUtensorMap tma,
                  const __grid_constant__ CUtensorMap tmb, const __grid_constant__ CUtensorMap tmal,
                  const __grid_constant__ CUtensorMap tmbl) {
  // F32: tma / tmb map the pre-split hi operands, tmal / tmbl the lo ones
  // (tf32_split_kernel); BF16 ignores tmal / tmbl.
  using C = Cfg<DT>;
  using L = MLayout<DT>;
  constexpr int BK = C::BK, STAGES = C::STAGES;
  extern __shared__ __align__(1024) char smem_raw[];
  char *smem = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * L::STAGE);
  uint64_t *empty = full + STAGES;
  uint64_t *tfull = empty + 2 * STAGES;      // (a reserved barrier slot per stage in between)
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  const int64_t ti0 = a.lb0 / BM, tj0 = a.lb1 / BN;
  const int64_t ntr = (a.ub0 + BM - 1) / BM - ti0, ntc = (a.ub1 + BN - 1) / BN - tj0;
  const int64_t nt = ntr * ntc;
  const int KB = (int)((a.K + BK - 1) / BK);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tma);
    tma_prefetch_desc(&tmb);
    for (int s = 0; s < STAGES; ++s) {
      tma_mbar_init(full + s, 1);
      tma_mbar_init(empty + s, 1);
    }
    for (int s = 0; s < 2; ++s) {
      tma_mbar_init(tfull + s, 1);
      tma_mbar_init(tempty + s, 4);
    }
    tma_fence_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tma_smem(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  TileSeq seq;
  seq.init(a.sched, a.chunk, nt);

  if (warp == 0) {
    if (lane == 0) {   // ---------------- TMA producer (operand tiles; F32: hi -> copy 0, lo -> copy 1)
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = seq.next(); tile >= 0; tile = seq.next()) {
        int64_t ti, tj;
        tile_coords(tile, ntr, ntc, ti, tj);
        const int m0 = (int)((ti0 + ti) * BM), n0 = (int)((tj0 + tj) * BN);
        for (int kb = 0; kb < KB; ++kb) {
          tma_mbar_wait(empty + stage, phase ^ 1);
          char *sa = smem + stage * L::STAGE;
          char *sb = sa + L::A_BYTES;
          tma_mbar_expect_tx(full + stage, L::TX);
          tma_load_2d(sa, &tma, kb * BK, m0 - (int)a.row0, full + stage);
#pragma unroll
          for (int j = 0; j < BN / L::BOXN; ++j)
            tma_load_2d(sb + j * L::B_BOX, &tmb, n0 + L::BOXN * j, kb * BK, full + stage);
          if constexpr (DT == UPIR_F32) {
            tma_load_2d(sa + L::COPY, &tmal, kb * BK, m0 - (int)a.row0, full + stage);
#pragma unroll
            for (int j = 0; j < BN / L::BOXN; ++j)
              tma_load_2d(sb + L::COPY + j * L::B_BOX, &tmbl, n0 + L::BOXN * j, kb * BK, full + stage);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {   // ---------------- MMA issuer
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int64_t tile = seq.next(); tile >= 0; tile = seq.next(), ++local) {
        const int acc = local & 1;
        const uint32_t acc_phase = (uint32_t)((local >> 1) & 1);
        tma_mbar_wait(tempty + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < KB; ++kb) {
          tma_mbar_wait(full + stage, phase);
          tc_fence_after();
          const char *hi = smem + stage * L::STAGE;
#pragma unroll
          for (int k = 0; k < BK / C::KSTEP; ++k) {
            // A K-major SW128: K step = 32 B inside the atom; SBO = 8 rows x 128 B.
            // B MN-major SW128: K step = KSTEP k-rows (x 128 B); LBO = box stride, SBO = 8 k-rows.
            // (MN-major tf32 must use SWIZZLE_128B_BASE32B: 32-B atoms, 4-row groups, SBO = 512 B.)
            constexpr uint64_t BLT = DT == UPIR_F32 ? LT_SW128_BASE32B : LT_SW128;
            constexpr uint32_t BSBO = DT == UPIR_F32 ? 512 : 1024;
            const uint64_t ah = smem_desc(hi + k * 32, 16, 1024);
            const uint64_t bh = smem_desc(hi + L::A_BYTES + k * C::KSTEP * 128, L::B_BOX, BSBO, BLT);
            if constexpr (DT == UPIR_BF16) {
              mma<DT>(tmem_d, ah, bh, (kb | k) != 0);
            } else {
              const char *lo = hi + L::COPY;
              const uint64_t al = smem_desc(lo + k * 32, 16, 1024);
              const uint64_t bl = smem_desc(lo + L::A_BYTES + k * C::KSTEP * 128, L::B_BOX, BSBO, BLT);
              mma<DT>(tmem_d, al, bh, (kb | k) != 0);   // lo_a * hi_b
              mma<DT>(tmem_d, ah, bl, 1);               // hi_a * lo_b
              mma<DT>(tmem_d, ah, bh, 1);               // hi_a * hi_b
            }
          }
          mma_commit(empty + stage);   // smem stage free once these MMAs complete
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        mma_commit(tfull + acc);   // accumulator ready
      }
    }
  } else if (warp >= 4 && warp < 8) {   // ---------------- epilogue
    const int ew = warp & 3;   // TMEM lanes [32*ew, 32*ew+32)
    int local = 0;
    for (int64_t tile = seq.next(); tile >= 0; tile = seq.next(), ++local) {
      const int acc = local & 1;
      const uint32_t acc_phase = (uint32_t)((local >> 1) & 1);
      int64_t ti, tj;
      tile_coords(tile, ntr, ntc, ti, tj);
      const int64_t m0 = (ti0 + ti) * BM, n0 = (tj0 + tj) * BN;
      tma_mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
      const int64_t row = m0 + 32 * ew + lane;
      const bool row_ok = row >= a.lb0 && row < a.ub0;
      float *crow = a.C + (row - a.row0) * a.ldc;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(32 * ew) << 16) + (uint32_t)(acc * BN + c), r);
        const int64_t col0 = n0 + c;
        if (!row_ok) continue;
        if (col0 >= a.lb1 && col0 + 32 <= a.ub1) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(crow + col0 + 8 * q),
                         "r"(r[8 * q]), "r"(r[8 * q + 1]), "r"(r[8 * q + 2]), "r"(r[8 * q + 3]), "r"(r[8 * q + 4]),
                         "r"(r[8 * q + 5]), "r"(r[8 * q + 6]), "r"(r[8 * q + 7])
                         : "memory");
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (col0 + q >= a.lb1 && col0 + q < a.ub1) crow[col0 + q] = __uint_as_float(r[q]);
        }
      }
      if (a.trace && ew == 0 && lane == 0) {
        a.trace[tile] = blockIdx.x;
        a.trace[nt + tile] = 0;
        atomicAdd(a.trace + 2 * nt + tile, 1);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) tma_mbar_arrive(tempty + acc);
    }
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(TMEM_COLS));
}

// ---------------------------------------------------------------------------
// CTA-pair variant (bf16): a TEAM is a cluster of 2 CTAs (reading c24: "team =
// the CTA pair when cta_group::2 is used"), 2 x 256 = 512 units.  The pair
// owns 256 x 256 output tiles: CTA r stages A rows [m0 + 128 r, +128) and B
// columns [n0 + 128 r, +128); the leader issues tcgen05.mma.cta_group::2
// (M = 256, N = 256) over both CTAs' shared memory; each CTA's TMEM receives
// its 128 rows.  Both CTAs' TMA loads complete on the LEADER's full barrier
// (cp.async.bulk.tensor ... .cta_group::2), MMA completion is multicast to
// both CTAs' empty / tmem-full barriers, and both epilogues release the
// accumulator on the leader's tmem-empty barrier.  B traffic per SM halves.
constexpr int PBM = 256, PSTAGES = 6;
constexpr int P_A = 128 * 64 * 2;              // this CTA's A rows
constexpr int P_B = 64 * 128 * 2;              // this CTA's B columns (2 boxes)
constexpr int P_STAGE = P_A + P_B;
constexpr int P_SMEM = PSTAGES * P_STAGE + 1024 + 256;
constexpr uint32_t P_IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) |
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(PBM >> 4) << 24);

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t map_to_cta(uint32_t smem_addr, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(smem_addr), "r"(cta));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ void tma_load_2d_pair(void *dst, const void *tmap, int c0, int c1, uint32_t bar_cluster) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], "
      "[%4];\n" ::"r"(tma_smem(dst)),
      "l"(tmap), "r"(c0), "r"(c1), "r"(bar_cluster)
      : "memory");
}
__device__ __forceinline__ void mma_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(P_IDESC), "r"(accum));
}
__device__ __forceinline__ void commit_pair(uint64_t *bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
          tma_smem(bar)),
      "h"((uint16_t)0x3)
      : "memory");
}
__device__ __forceinline__ void remote_arrive(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];\n" ::"r"(bar_cluster) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1)
    matmul_pair_kernel(const __grid_constant__ MatmulArgs a, const __grid_constant__ CUtensorMap tma,
                       const __grid_constant__ CUtensorMap tmb) {
  extern __shared__ __align__(1024) char smem_raw[];
  char *smem = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + PSTAGES * P_STAGE);
  uint64_t *empty = full + PSTAGES;
  uint64_t *tfull = empty + PSTAGES;
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;

  const int64_t ti0 = a.lb0 / PBM, tj0 = a.lb1 / BN;
  const int64_t ntr = (a.ub0 + PBM - 1) / PBM - ti0, ntc = (a.ub1 + BN - 1) / BN - tj0;
  const int64_t nt = ntr * ntc;
  const int KB = (int)((a.K + 64 - 1) / 64);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tma);
    tma_prefetch_desc(&tmb);
    for (int st = 0; st < PSTAGES; ++st) {
      tma_mbar_init(full + st, 1);
      tma_mbar_init(empty + st, 1);
    }
    for (int st = 0; st < 2; ++st) {
      tma_mbar_init(tfull + st, 1);
      tma_mbar_init(tempty + st, 8);   // 4 epilogue warps x 2 CTAs (leader's copy is used)
    }
    tma_fence_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tma_smem(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  // the pair's tile sequence (teams = pairs)
  TileSeq seq;
  {
    seq.sched = a.sched;
    seq.chunk = a.chunk;
    seq.nt = nt;
    seq.p = gridDim.x / 2;
    seq.t = blockIdx.x / 2;
    if (seq.sched == SK_STATIC_BLOCK) {
      const int64_t q = nt / seq.p, r = nt % seq.p;
      seq.cur = seq.t * q + (seq.t < r ? seq.t : r);
      seq.end = seq.cur + q + (seq.t < r ? 1 : 0);
      seq.k = 0;
    } else {
      seq.k = seq.t;
      seq.cur = seq.k * seq.chunk;
      seq.end = min(nt, seq.cur + seq.chunk);
    }
  }

  if (warp == 0) {
    if (lane == 0) {   // ---------------- TMA producer (both CTAs)
      const uint32_t full_leader = map_to_cta(tma_smem(full), 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = seq.next(); tile >= 0; tile = seq.next()) {
        int64_t ti, tj;
        tile_coords(tile, ntr, ntc, ti, tj);
        const int m0 = (int)((ti0 + ti) * PBM + 128 * rank), n0 = (int)((tj0 + tj) * BN + 128 * rank);
        for (int kb = 0; kb < KB; ++kb) {
          tma_mbar_wait(empty + stage, phase ^ 1);
          char *sa = smem + stage * P_STAGE;
          char *sb = sa + P_A;
          if (leader) tma_mbar_expect_tx(full + stage, 2 * P_STAGE);
          const uint32_t fb = full_leader + (uint32_t)(stage * 8);
          tma_load_2d_pair(sa, &tma, kb * 64, m0 - (int)a.row0, fb);
          tma_load_2d_pair(sb, &tmb, n0, kb * 64, fb);
          tma_load_2d_pair(sb + 8192, &tmb, n0 + 64, kb * 64, fb);
          if (++stage == PSTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {   // ---------------- MMA issuer (leader CTA only)
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int64_t tile = seq.next(); tile >= 0; tile = seq.next(), ++local) {
        const int acc = local & 1;
        const uint32_t acc_phase = (uint32_t)((local >> 1) & 1);
        tma_mbar_wait(tempty + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < KB; ++kb) {
          tma_mbar_wait(full + stage, phase);
          tc_fence_after();
          const char *sa = smem + stage * P_STAGE;
          const char *sb = sa + P_A;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ad = smem_desc(sa + k * 32, 16, 1024);
            const uint64_t bd = smem_desc(sb + k * 2048, 8192, 1024);
            mma_pair(tmem_d, ad, bd, (kb | k) != 0);
          }
          commit_pair(empty + stage);   // both CTAs' smem stages free
          if (++stage == PSTAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        commit_pair(tfull + acc);   // both CTAs' accumulators ready
      }
    }
  } else if (warp >= 4) {   // ---------------- epilogue (both CTAs)
    const int ew = warp & 3;
    const uint32_t tempty_leader = map_to_cta(tma_smem(tempty), 0);
    int local = 0;
    for (int64_t tile = seq.next(); tile >= 0; tile = seq.next(), ++local) {
      const int acc = local & 1;
      const uint32_t acc_phase = (uint32_t)((local >> 1) & 1);
      int64_t ti, tj;
      tile_coords(tile, ntr, ntc, ti, tj);
      const int64_t m0 = (ti0 + ti) * PBM + 128 * rank, n0 = (tj0 + tj) * BN;
      tma_mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
      const int64_t row = m0 + 32 * ew + lane;
      const bool row_ok = row >= a.lb0 && row < a.ub0;
      float *crow = a.C + (row - a.row0) * a.ldc;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(32 * ew) << 16) + (uint32_t)(acc * BN + c), r);
        const int64_t col0 = n0 + c;
        if (!row_ok) continue;
        if (col0 >= a.lb1 && col0 + 32 <= a.ub1) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(crow + col0 + 8 * q),
                         "r"(r[8 * q]), "r"(r[8 * q + 1]), "r"(r[8 * q + 2]), "r"(r[8 * q + 3]), "r"(r[8 * q + 4]),
                         "r"(r[8 * q + 5]), "r"(r[8 * q + 6]), "r"(r[8 * q + 7])
                         : "memory");
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (col0 + q >= a.lb1 && col0 + q < a.ub1) crow[col0 + q] = __uint_as_float(r[q]);
        }
      }
      if (a.trace && leader && ew == 0 && lane == 0) {
        a.trace[tile] = (int32_t)(blockIdx.x / 2);
        a.trace[nt + tile] = 0;
        atomicAdd(a.trace + 2 * nt + tile, 1);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) remote_arrive(tempty_leader + (uint32_t)(acc * 8));
    }
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(TMEM_COLS));
}

// CTA-pair variant for fp32 inputs (3xTF32): a team = 2 CTAs x 384 units.
// The operands arrive pre-split (tf32_split_kernel: hi = rna_tf32(x),
// lo = x - hi, one elementwise pass over A and B before the loop kernel), so
// both CTAs' TMA loads of the hi and lo tiles (.cta_group::2) complete on
// the LEADER's full barrier and no shared-memory rewrite competes with the
// tensor core for shared-memory bandwidth; the leader issues
// tcgen05.mma.cta_group::2.kind::tf32 (M = 256, N = 256, K = 8) three times
// per k-step.  3 stages of 64 KB (hi + lo of A and B halves) per CTA.
// Warps 8..11 of the 384-unit team have no role in this variant.
constexpr int PF_STAGES = 3;
constexpr int PF_A = 128 * 32 * 4;            // 16 KB: this CTA's A rows (one copy)
constexpr int PF_B = 32 * 128 * 4;            // 16 KB: this CTA's B columns (4 boxes of 32)
constexpr int PF_COPY = PF_A + PF_B;
constexpr int PF_STAGE = 2 * PF_COPY;
constexpr int PF_SMEM = PF_STAGES * PF_STAGE + 1024 + 256;
constexpr uint32_t PF_IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (0u << 15) | (1u << 16) |
                              ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(PBM >> 4) << 24);

__device__ __forceinline__ void mma_pair_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t accum) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(PF_IDESC), "r"(accum));
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    matmul_pair_f32_kernel(const __grid_constant__ MatmulArgs a, const __grid_constant__ CUtensorMap tma,
                           const __grid_constant__ CUtensorMap tmb, const __grid_constant__ CUtensorMap tmal,
                           const __grid_constant__ CUtensorMap tmbl) {
  extern __shared__ __align__(1024) char smem_raw[];
  char *smem = reinterpret_cast<char *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~(uintptr_t)1023);
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + PF_STAGES * PF_STAGE);
  uint64_t *empty = full + PF_STAGES;
  uint64_t *tfull = empty + 2 * PF_STAGES;   // (a reserved barrier slot per stage in between)
  uint64_t *tempty = tfull + 2;
  uint32_t *tmem_holder = reinterpret_cast<uint32_t *>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;

  const int64_t ti0 = a.lb0 / PBM, tj0 = a.lb1 / BN;
  const int64_t ntr = (a.ub0 + PBM - 1) / PBM - ti0, ntc = (a.ub1 + BN - 1) / BN - tj0;
  const int64_t nt = ntr * ntc;
  const int KB = (int)((a.K + 32 - 1) / 32);

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tma);
    tma_prefetch_desc(&tmb);
    tma_prefetch_desc(&tmal);
    tma_prefetch_desc(&tmbl);
    for (int st = 0; st < PF_STAGES; ++st) {
      tma_mbar_init(full + st, 1);
      tma_mbar_init(empty + st, 1);
    }
    for (int st = 0; st < 2; ++st) {
      tma_mbar_init(tfull + st, 1);
      tma_mbar_init(tempty + st, 8);
    }
    tma_fence_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tma_smem(tmem_holder)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_holder;

  TileSeq seq;
  seq.sched = a.sched;
  seq.chunk = a.chunk;
  seq.nt = nt;
  seq.p = gridDim.x / 2;
  seq.t = blockIdx.x / 2;
  if (seq.sched == SK_STATIC_BLOCK) {
    const int64_t q = nt / seq.p, r = nt % seq.p;
    seq.cur = seq.t * q + (seq.t < r ? seq.t : r);
    seq.end = seq.cur + q + (seq.t < r ? 1 : 0);
    seq.k = 0;
  } else {
    seq.k = seq.t;
    seq.cur = seq.k * seq.chunk;
    seq.end = min(nt, seq.cur + seq.chunk);
  }

  if (warp == 0) {
    if (lane == 0) {   // ---------------- TMA producer (both CTAs -> the leader's full barrier)
      const uint32_t full_leader = map_to_cta(tma_smem(full), 0);
      int stage = 0;
      uint32_t phase = 0;
      for (int64_t tile = seq.next(); tile >= 0; tile = seq.next()) {
        int64_t ti, tj;
        tile_coords(tile, ntr, ntc, ti, tj);
        const int m0 = (int)((ti0 + ti) * PBM + 128 * rank), n0 = (int)((tj0 + tj) * BN + 128 * rank);
        for (int kb = 0; kb < KB; ++kb) {
          tma_mbar_wait(empty + stage, phase ^ 1);
          char *sa = smem + stage * PF_STAGE;   // hi copy: A, B; lo copy at + PF_COPY
          char *sb = sa + PF_A;
          if (leader) tma_mbar_expect_tx(full + stage, 2 * PF_STAGE);
          const uint32_t fb = full_leader + (uint32_t)(stage * 8);
          tma_load_2d_pair(sa, &tma, kb * 32, m0 - (int)a.row0, fb);
          tma_load_2d_pair(sa + PF_COPY, &tmal, kb * 32, m0 - (int)a.row0, fb);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            tma_load_2d_pair(sb + j * 4096, &tmb, n0 + 32 * j, kb * 32, fb);
            tma_load_2d_pair(sb + PF_COPY + j * 4096, &tmbl, n0 + 32 * j, kb * 32, fb);
          }
          if (++stage == PF_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && leader) {   // ---------------- MMA issuer (leader)
      int stage = 0;
      uint32_t phase = 0;
      int local = 0;
      for (int64_t tile = seq.next(); tile >= 0; tile = seq.next(), ++local) {
        const int acc = local & 1;
        const uint32_t acc_phase = (uint32_t)((local >> 1) & 1);
        tma_mbar_wait(tempty + acc, acc_phase ^ 1);
        tc_fence_after();
        const uint32_t tmem_d = tmem_base + (uint32_t)(acc * BN);
        for (int kb = 0; kb < KB; ++kb) {
          tma_mbar_wait(full + stage, phase);
          tc_fence_after();
          const char *hi = smem + stage * PF_STAGE;
          const char *lo = hi + PF_COPY;
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const uint64_t ah = smem_desc(hi + k * 32, 16, 1024);
            const uint64_t al = smem_desc(lo + k * 32, 16, 1024);
            const uint64_t bh = smem_desc(hi + PF_A + k * 1024, 4096, 512, LT_SW128_BASE32B);
            const uint64_t bl = smem_desc(lo + PF_A + k * 1024, 4096, 512, LT_SW128_BASE32B);
            mma_pair_tf32(tmem_d, al, bh, (kb | k) != 0);   // lo_a * hi_b
            mma_pair_tf32(tmem_d, ah, bl, 1);               // hi_a * lo_b
            mma_pair_tf32(tmem_d, ah, bh, 1);               // hi_a * hi_b
          }
          commit_pair(empty + stage);
          if (++stage == PF_STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        commit_pair(tfull + acc);
      }
    }
  } else if (warp >= 4 && warp < 8) {   // ---------------- epilogue (both CTAs)
    const int ew = warp & 3;
    const uint32_t tempty_leader = map_to_cta(tma_smem(tempty), 0);
    int local = 0;
    for (int64_t tile = seq.next(); tile >= 0; tile = seq.next(), ++local) {
      const int acc = local & 1;
      const uint32_t acc_phase = (uint32_t)((local >> 1) & 1);
      int64_t ti, tj;
      tile_coords(tile, ntr, ntc, ti, tj);
      const int64_t m0 = (ti0 + ti) * PBM + 128 * rank, n0 = (tj0 + tj) * BN;
      tma_mbar_wait(tfull + acc, acc_phase);
      tc_fence_after();
      const int64_t row = m0 + 32 * ew + lane;
      const bool row_ok = row >= a.lb0 && row < a.ub0;
      float *crow = a.C + (row - a.row0) * a.ldc;
#pragma unroll 1
      for (int c = 0; c < BN; c += 32) {
        uint32_t r[32];
        tmem_ld32(tmem_base + ((uint32_t)(32 * ew) << 16) + (uint32_t)(acc * BN + c), r);
        const int64_t col0 = n0 + c;
        if (!row_ok) continue;
        if (col0 >= a.lb1 && col0 + 32 <= a.ub1) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(crow + col0 + 8 * q),
                         "r"(r[8 * q]), "r"(r[8 * q + 1]), "r"(r[8 * q + 2]), "r"(r[8 * q + 3]), "r"(r[8 * q + 4]),
                         "r"(r[8 * q + 5]), "r"(r[8 * q + 6]), "r"(r[8 * q + 7])
                         : "memory");
        } else {
#pragma unroll
          for (int q = 0; q < 32; ++q)
            if (col0 + q >= a.lb1 && col0 + q < a.ub1) crow[col0 + q] = __uint_as_float(r[q]);
        }
      }
      if (a.trace && leader && ew == 0 && lane == 0) {
        a.trace[tile] = (int32_t)(blockIdx.x / 2);
        a.trace[nt + tile] = 0;
        atomicAdd(a.trace + 2 * nt + tile, 1);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) remote_arrive(tempty_leader + (uint32_t)(acc * 8));
    }
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  if (warp == 2)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_base), "r"(TMEM_COLS));
}

// 3xTF32 operand split (pair variant): hi = rna_tf32(x), lo = x - hi, over
// n elements (16-B vectors, scalar tail).
__global__ void tf32_split_kernel(const float *__restrict__ src, float *__restrict__ hi, float *__restrict__ lo,
                                  int64_t n) {
  const int64_t n4 = n / 4, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const float4 x = __ldcs(reinterpret_cast<const float4 *>(src) + i);
    float4 h, l;
    h.x = to_tf32(x.x);
    h.y = to_tf32(x.y);
    h.z = to_tf32(x.z);
    h.w = to_tf32(x.w);
    l.x = __fsub_rn(x.x, h.x);
    l.y = __fsub_rn(x.y, h.y);
    l.z = __fsub_rn(x.z, h.z);
    l.w = __fsub_rn(x.w, h.w);
    reinterpret_cast<float4 *>(hi)[i] = h;
    reinterpret_cast<float4 *>(lo)[i] = l;
  }
  for (int64_t i = 4 * n4 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const float h = to_tf32(src[i]);
    hi[i] = h;
    lo[i] = __fsub_rn(src[i], h);
  }
}

}  // namespace

cudaError_t launch_tf32_split(const float *src, float *hi, float *lo, int64_t n, int num_sms, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const int64_t blocks = std::min<int64_t>((int64_t)num_sms * 4, (n / 4 + 255) / 256 + 1);
  tf32_split_kernel<<<(int)blocks, 256, 0, s>>>(src, hi, lo, n);
  return cudaGetLastError();
}
bool matmul_f32_presplit(int) { return true; }   // both fp32 variants stream pre-split operands

int matmul_tile_m() { return BM; }
int matmul_tile_n() { return BN; }
int matmul_required_units(int dtype) { return dtype == UPIR_F32 ? Cfg<UPIR_F32>::THREADS : Cfg<UPIR_BF16>::THREADS; }
// bf16 teams may also be CTA pairs (512 units, 256-row tiles)
bool matmul_units_ok(int dtype, int units) {
  return units == matmul_required_units(dtype) || (dtype == UPIR_BF16 && units == 512) ||
         (dtype == UPIR_F32 && units == 768);
}
int matmul_tile_m_for(int dtype, int units) {
  return ((dtype == UPIR_BF16 && units == 512) || (dtype == UPIR_F32 && units == 768)) ? PBM : BM;
}

bool matmul_encode_tmaps(void *tma, void *tmb, const void *A, const void *B, int dtype, int64_t M, int64_t N,
                         int64_t K, int64_t lda, int64_t ldb) {
  const bool f32 = dtype == UPIR_F32;
  const CUtensorMapDataType dt = f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const int es = f32 ? 4 : 2, bk = f32 ? Cfg<UPIR_F32>::BK : Cfg<UPIR_BF16>::BK, boxn = 128 / es;
  return encode_tmap_2d(reinterpret_cast<CUtensorMap *>(tma), dt, A, (uint64_t)K, (uint64_t)M, (uint64_t)lda * es,
                        bk, BM, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B) &&
         encode_tmap_2d(reinterpret_cast<CUtensorMap *>(tmb), dt, B, (uint64_t)N, (uint64_t)K, (uint64_t)ldb * es,
                        boxn, bk, f32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B);
}

template <int DT>
static cudaError_t launch_dt(const MatmulArgs &a, int teams, cudaStream_t s) {
  using L = MLayout<DT>;
  cudaError_t e = cudaFuncSetAttribute(matmul_kernel<DT>, cudaFuncAttributeMaxDynamicSharedMemorySize, L::SMEM);
  if (e != cudaSuccess) return e;
  const CUtensorMap &ta = *reinterpret_cast<const CUtensorMap *>(a.tmap_a);
  const CUtensorMap &tb = *reinterpret_cast<const CUtensorMap *>(a.tmap_b);
  if (DT == UPIR_F32 && (!a.tmap_a2 || !a.tmap_b2)) return cudaErrorInvalidValue;   // needs the pre-split lo operands
  const CUtensorMap &ta2 = DT == UPIR_F32 ? *reinterpret_cast<const CUtensorMap *>(a.tmap_a2) : ta;
  const CUtensorMap &tb2 = DT == UPIR_F32 ? *reinterpret_cast<const CUtensorMap *>(a.tmap_b2) : tb;
  matmul_kernel<DT><<<teams, Cfg<DT>::THREADS, L::SMEM, s>>>(a, ta, tb, ta2, tb2);
  return cudaGetLastError();
}

cudaError_t launch_matmul(const MatmulArgs &a, int dtype, int teams, int units, cudaStream_t s) {
  if (dtype == UPIR_BF16 && units == 512) {
    cudaError_t e = cudaFuncSetAttribute(matmul_pair_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM);
    if (e != cudaSuccess) return e;
    matmul_pair_kernel<<<2 * teams, 256, P_SMEM, s>>>(a, *reinterpret_cast<const CUtensorMap *>(a.tmap_a),
                                                     *reinterpret_cast<const CUtensorMap *>(a.tmap_b));
    return cudaGetLastError();
  }
  if (dtype == UPIR_F32 && units == 768) {
    cudaError_t e = cudaFuncSetAttribute(matmul_pair_f32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, PF_SMEM);
    if (e != cudaSuccess) return e;
    if (!a.tmap_a2 || !a.tmap_b2) return cudaErrorInvalidValue;   // needs the pre-split lo operands
    matmul_pair_f32_kernel<<<2 * teams, 384, PF_SMEM, s>>>(a, *reinterpret_cast<const CUtensorMap *>(a.tmap_a),
                                                          *reinterpret_cast<const CUtensorMap *>(a.tmap_b),
                                                          *reinterpret_cast<const CUtensorMap *>(a.tmap_a2),
                                                          *reinterpret_cast<const CUtensorMap *>(a.tmap_b2));
    return cudaGetLastError();
  }
  if (units != matmul_required_units(dtype)) return cudaErrorInvalidValue;
  if (dtype == UPIR_BF16) return launch_dt<UPIR_BF16>(a, teams, s);
  if (dtype == UPIR_F32) return launch_dt<UPIR_F32>(a, teams, s);
  return cudaErrorInvalidValue;
}

}  // namespace upir
