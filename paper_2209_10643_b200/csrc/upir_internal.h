// upir_internal.h -- shared declarations between the runtime (upir_runtime.cu)
// and the kernel translation units.  Not part of the C-ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/upir.h"

namespace upir {

// Schedule kinds after host-side resolution (readings c3-c8).
enum SchedKind : int32_t { SK_STATIC_BLOCK = 0, SK_STATIC_CHUNK = 1, SK_DYNAMIC = 2, SK_GUIDED = 3 };

// Memory path of the 1-D streaming kernels.
enum PathKind : int32_t {
  PATH_DIRECT = 0,   // each unit loads its own elements (small chunks: coalesced)
  PATH_STAGED = 1    // warp-cooperative cp.async staging of 128/64-B unit segments
};

// ---- peer window (one per context; exported to the other ranks by CUDA IPC) --
// 64-bit words.  Remote ranks write the counters / slots of THIS window over
// NVLink; the peer table holds this rank's mapped pointers to every rank's
// window (entry `rank` = the local window).
enum WinWord : int32_t {
  WIN_HALO_FROM_UP = 0,   // sweeps delivered by rank - 1 (monotonic)
  WIN_HALO_FROM_DN = 1,   // sweeps delivered by rank + 1
  WIN_HALO_GEN = 2,       // peer-mode sweeps this rank completed
  WIN_HALO_DONE = 3,      // last-team ticket of a peer-mode sweep
  WIN_WR_CNT = 8,         // world-reduce arrivals (monotonic, N per reduction)
  WIN_WR_GEN = 9,         // world reductions this rank completed
  WIN_BAR_CNT = 10,       // peer-barrier arrivals (monotonic, N per barrier)
  WIN_BAR_GEN = 11,       // peer barriers this rank completed
  WIN_AR_CNT = 12,        // peer-allreduce arrivals (monotonic, N per upir_reduce(WORLD))
  WIN_AR_GEN = 13,        // peer allreduces this rank completed
  WIN_WR_SLOTS = 16,      // [2 parity][WIN_MAX_RANKS][2 reductions] partials
  WIN_PEERS = 512,        // [WIN_MAX_RANKS] mapped window pointers
  WIN_WORDS = 576
};
constexpr int WIN_MAX_RANKS = 64;
// after the 8 KiB of words: the allreduce staging, [2 parity][WIN_AR_ELEMS] x 8 B
constexpr size_t WIN_AR_OFF = 8192;
constexpr int64_t WIN_AR_ELEMS = 65536;
constexpr size_t WIN_BYTES = WIN_AR_OFF + 2 * (size_t)WIN_AR_ELEMS * 8;
// upir_reduce(WORLD) over the peer windows (count <= WIN_AR_ELEMS): one CTA
// stages dev_in in its window, publishes to every rank, waits for all, and
// combines the ranks' staged values in ascending rank order.
cudaError_t launch_peer_allreduce(unsigned long long *win, int nranks, int op, int dtype, const void *dev_in,
                                  int64_t count, void *dev_out, cudaStream_t s);

// Streaming bodies.
enum StreamBody : int32_t { SB_RED_I64 = 0, SB_RED_F32 = 1, SB_AXPY = 2 };

struct RedSpec {
  int32_t op;           // upir_op
  int32_t dtype;        // UPIR_I64 / UPIR_F32
  uint64_t init_bits;   // init value: int64 bits, or fp64 bits for F32
  void *result;         // device scalar of dtype
};

// Arguments of the 1-D streaming loop kernels (axpy / reduce).
struct StreamArgs {
  // normalised iteration space: iteration k in [0,T) -> element i = lb + k*step
  int64_t T, lb, step;
  // schedule
  int32_t sched;        // SchedKind
  int32_t distribute;   // upir_distribute
  int64_t chunk;        // static-chunk / dynamic chunk size (iterations)
  int64_t ticket_m;     // dynamic: chunks per unit per ticket
  unsigned long long *dyn_counter;  // dynamic / guided: chunk counter (reset by the last team)
  const int64_t *gtab;  // guided: chunk boundaries b_0 = 0 < b_1 < ... < b_nc = T (nc + 1 entries)
  int64_t gchunks;      // guided: nc
  // body (pointers already shifted so that element i lives at ptr[i])
  const void *in0;      // reduce: data; axpy: x
  void *out;            // axpy: y
  float alpha;
  int64_t safe_lo, safe_hi;  // elements [safe_lo, safe_hi) may be read as 16-B vectors
  int32_t dvar;              // DIRECT long-chunk load variant (0: 4x16 B, 1: 4x32 B, 2: 2x32 B, 3: 8x16 B)
  // address alignment of the element views: element e lives at a 128-B
  // aligned base + (e + esh) * esz (esh < 128 / esz, identical for x and y);
  // vecok = 0 when x and y disagree (only scalar accesses are then legal)
  int32_t esh, vecok;
  int64_t simd;              // static block: SIMD group size (simdlen, reading c33), 1 = none
  // reductions
  int32_t nred;
  RedSpec red[2];
  unsigned long long *slots;   // [gridDim.x][2] team partials (8-byte words)
  unsigned int *done;          // last-team ticket (self-resetting)
  // world reduction fused into the epilogue (UPIR_WORLD_REDUCE): local peer
  // window or null; the last team combines init (+) P_0 (+) ... (+) P_{N-1}
  unsigned long long *wwin;
  int32_t wrank, wranks;
  // world reduction by a communicator instead: the last team writes the
  // rank's partials (int64 / fp64 bits, init NOT applied) here, for the
  // all-gather and the ordered fp64 combine (launch_world_combine)
  unsigned long long *wpart;
  // trace: [team[T], unit[T], hits[T]] int32, or null
  int32_t *trace;
};

// Launch helpers (defined in the kernel TUs).  Return cudaError_t.
cudaError_t launch_stream_loop(int body, int path, int segv, int nst, bool trace,
                               int teams, int units, size_t smem, const StreamArgs &a,
                               cudaStream_t s);
// Dynamic smem a staged config needs per CTA.
size_t staged_smem_bytes(int body, int units, int segv, int nst);

// Standalone device reduction of `count` elements (upir_reduce DEVICE) and
// the ordered combine of gathered per-rank partials (upir_reduce WORLD).
cudaError_t launch_reduce_array(int op, int dtype, const void *in, int64_t count, void *out,
                                unsigned long long *slots, unsigned int *done, cudaStream_t s);
// Peer mode: wait until both neighbours delivered every sweep this rank
// completed (before a peer-attached buffer is read back or released).
cudaError_t launch_peer_drain(unsigned long long *win, int has_up, int has_dn, cudaStream_t s);
// Barrier over all ranks through the peer windows (communicator-less worlds).
cudaError_t launch_peer_barrier(unsigned long long *win, int nranks, cudaStream_t s);
// upir_sync(HALO) over peer mappings: store my boundary rows [src, src +
// bytes) into the neighbours' halo rows (dst), publish, wait for theirs.
struct PeerHaloArgs {
  unsigned long long *win, *win_up, *win_dn;   // my window, neighbours' windows (null: none)
  const char *src_up, *src_dn;                 // my rows sent to rank - 1 / rank + 1
  char *dst_up, *dst_dn;                       // their halo rows (peer mappings)
  int64_t bytes_up, bytes_dn;
};
cudaError_t launch_peer_halo(const PeerHaloArgs &a, cudaStream_t s);
// result_r = init_r (+) g[0][r] (+) ... (+) g[nranks-1][r] over gathered
// [nranks][2] partial words of a loop's reductions (int64, or fp64 rounded once).
cudaError_t launch_world_combine(const unsigned long long *gathered, int nranks, int nred, const RedSpec *reds,
                                 cudaStream_t s);
cudaError_t launch_rank_combine(int op, int dtype, const void *gathered, int64_t count,
                                int nranks, void *out, cudaStream_t s);

// Synthetic fill (counter-based splitmix64).
cudaError_t launch_synth_fill(int dist, uint64_t stream, void *dst, int64_t n, int64_t index0,
                              int64_t n_rows, int64_t n_cols, cudaStream_t s);

// ---- Jacobi 5-point ----------------------------------------------------------
struct JacobiArgs {
  float *out;           // element (i, j) at out[(i - row0) * ld + j]
  int64_t ld;           // row pitch (elements)
  int64_t row0;         // global row of the first local row
  // iteration space (global induction values) [lb0,ub0) x [lb1,ub1), step 1
  int64_t lb0, ub0, lb1, ub1;
  // tiles anchored at 0: tile (ti, tj) = rows [ti*BM, +BM) x cols [tj*BN, +BN)
  int64_t ti0, tj0;     // first tile indices touching the space
  int64_t ntr, ntc;     // tile grid extent; tile id = (ti-ti0)*ntc + (tj-tj0)
  int32_t sched;        // tile loop over teams (SchedKind)
  int32_t inner_chunk;  // intra-tile static chunk over units
  int64_t chunk;
  unsigned long long *dyn_counter;
  unsigned int *done;
  int32_t *trace;       // [team | unit | hits] planes of ntiles*BM*BN int32, or null
  int32_t units;        // num_units (set by the launcher; the CTA may carry a producer warp)
  int32_t colmajor;     // tile ids column-major (UPIR_TILE_COLMAJOR, reading c35)
  int32_t reverse;      // tile ids from the last tile (UPIR_TILE_REVERSE)
  // fused halo exchange with ranks r-1 / r+1 (peer mode): null win = off
  unsigned long long *win;          // local peer window
  unsigned long long *win_up, *win_dn;  // neighbours' windows (null at the ends)
  float *peer_up, *peer_dn;         // neighbours' OUT buffers (local row 0)
  int64_t peer_up_row0, peer_dn_row0;
  int64_t send_up_row, send_dn_row;  // my first / last owned row (-1: none)
  int64_t halo_up_row, halo_dn_row;  // my halo rows read from the neighbours (-1: none)
};
bool jacobi_supported_tile(int bm, int bn);
// tmc / tmh: CUtensorMap (128 B) of the input buffer with boxes {BN, BM+2}
// and {4, BM+2}.
cudaError_t launch_jacobi_tma(const JacobiArgs &a, const void *tmc, const void *tmh, int teams, int units, int bm,
                              int bn, bool trace, cudaStream_t s);

// ---- 2-D filter stencil (NEXT #4) ---------------------------------------------------
struct StencilArgs {
  const float *in, *w;
  float *out;
  int64_t ld, row0, ny, nx;
  int64_t lb0, ub0, lb1, ub1;
  int64_t ti0, tj0, ntr, ntc;
  int32_t sched, inner_chunk;
  int64_t chunk;
  unsigned long long *dyn_counter;
  unsigned int *done;
  int32_t *trace;
  int32_t units;        // units per team (the launch may add a producer warp)
};
bool stencil_supported(int F, int bm, int bn);
cudaError_t launch_stencil(const StencilArgs &a, int F, int bm, int bn, int teams, int units, cudaStream_t s);

// ---- matvec (NEXT #2) -------------------------------------------------------------
struct MatvecArgs {
  const float *A, *x;
  float *y;
  int64_t K, lda;
  int64_t lb, T;                // rows [lb, lb + T)
  int32_t sched, distribute;
  int64_t chunk;
  int32_t inner_chunk;
  unsigned long long *dyn_counter;
  unsigned int *done;
  int32_t *trace;               // [team | unit | hits] x T, or null
  int64_t simd;                 // static block over SIMD groups of this many rows (1 = none)
};
cudaError_t launch_matvec(const MatvecArgs &a, int teams, int units, cudaStream_t s);

// ---- matmul (tcgen05) ------------------------------------------------------------
struct MatmulArgs {
  const void *A, *B;
  float *C;
  int64_t M, N, K, lda, ldb, ldc;
  int64_t lb0, ub0, lb1, ub1;   // (i, j) iteration space (global rows)
  int64_t row0;                 // global row of local row 0 of A and C (BLOCK maps)
  int32_t sched;
  int64_t chunk;
  int64_t ticket_m;
  unsigned long long *dyn_counter;
  int32_t *trace;               // tile -> team owner (tile granularity) or null
  void *tmap_a, *tmap_b;        // host CUtensorMaps (passed by value at launch)
  void *tmap_a2, *tmap_b2;      // 3xTF32 pair variant: maps of the pre-split lo operands (a/b = hi)
};
// 3xTF32 pre-split of an fp32 operand (pair variant): hi = rna_tf32(x), lo = x - hi.
cudaError_t launch_tf32_split(const float *src, float *hi, float *lo, int64_t n, int num_sms, cudaStream_t s);
bool matmul_f32_presplit(int units);
cudaError_t launch_matmul(const MatmulArgs &a, int dtype, int teams, int units, cudaStream_t s);
bool matmul_encode_tmaps(void *tma, void *tmb, const void *A, const void *B, int dtype,
                         int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb);
int matmul_tile_m();
int matmul_tile_n();
int matmul_required_units(int dtype);
bool matmul_units_ok(int dtype, int units);
int matmul_tile_m_for(int dtype, int units);

}  // namespace upir
