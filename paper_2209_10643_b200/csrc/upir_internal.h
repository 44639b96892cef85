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
  // reductions
  int32_t nred;
  RedSpec red[2];
  unsigned long long *slots;   // [gridDim.x][2] team partials (8-byte words)
  unsigned int *done;          // last-team ticket (self-resetting)
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
};
cudaError_t launch_matmul(const MatmulArgs &a, int dtype, int teams, int units, cudaStream_t s);
bool matmul_encode_tmaps(void *tma, void *tmb, const void *A, const void *B, int dtype,
                         int64_t M, int64_t N, int64_t K, int64_t lda, int64_t ldb);
int matmul_tile_m();
int matmul_tile_n();
int matmul_required_units(int dtype);
bool matmul_units_ok(int dtype, int units);
int matmul_tile_m_for(int dtype, int units);

}  // namespace upir
