/*
 * upir.h -- C-ABI of the B200-native UPIR data-parallel loop runtime.
 *
 * Executes a lowered UPIR data-parallel loop nest (arXiv 2209.10643): an SPMD
 * region of teams x units (Fig. 1 `upir.spmd`) running a
 * worksharing `upir.loop` (Fig. 3) under a schedule, with
 * `upir.sync reduction / allreduce / send / recv / barrier` (PAPER.md:867-898,
 * Fig. 7) and explicit `upir.data` mapping and movement (PAPER.md:736-865,
 * Figs. 5-6).  The call set follows the lowered runtime primitives of
 * SPEC.md:294-299 (fork_teams/fork_units -> upir_spmd_launch, dispatch_loop ->
 * upir_loop_exec, reduce -> upir_reduce, barrier -> upir_sync,
 * map_enter/map_exit/alloc/dealloc/memcpy -> upir_data_*).
 *
 * Conventions (all entry points):
 *  - Every call returns upir_status.  Out-params are written only on UPIR_OK.
 *  - Descriptors are validated BEFORE anything is enqueued: an invalid call has
 *    no side effect.  upir_last_error() returns a thread-local message.
 *  - Asynchronous CUDA/NCCL failures are sticky on the context and are
 *    reported by the next upir_sync / upir_data_unmap / upir_finalize.
 *  - Geometry is honoured exactly or rejected with UPIR_E_INVALID, never
 *    clamped (lesson of PAPER.md:1578-1587: GCC clamps to 256 threads).
 *  - All iteration arithmetic is int64 (T = 2^34 at 8 GPUs).
 *  - Host pointers stay caller-owned; device memory of a map is owned by the
 *    context's present table (refcounted) unless adopted.
 *  - One host thread per context.  No C++ exception crosses this ABI.
 *  - There is no CPU fallback: without a usable sm_100 device upir_init fails.
 */
#ifndef UPIR_H
#define UPIR_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status ----------------------------------------------------------- */
typedef enum {
    UPIR_OK = 0,
    UPIR_E_INVALID = 1,     /* bad descriptor / geometry / argument           */
    UPIR_E_UNSUPPORTED = 2, /* valid UPIR, not implemented (e.g. taskloop)      */
    UPIR_E_NOT_MAPPED = 3,  /* body names a buffer absent from the present table */
    UPIR_E_OOM = 4,
    UPIR_E_CUDA = 5,
    UPIR_E_NCCL = 6,
    UPIR_E_SYNC = 7,        /* wait without arrive / mismatched async pair      */
    UPIR_E_LEAK = 8         /* finalize with live maps                          */
} upir_status;

/* Thread-local message for the last non-OK status of this thread. */
const char *upir_last_error(void);
/* Library version string. */
const char *upir_version(void);

typedef enum { UPIR_I32 = 0, UPIR_I64 = 1, UPIR_F32 = 2, UPIR_F64 = 3, UPIR_BF16 = 4 } upir_dtype;

typedef struct upir_ctx_s *upir_ctx;
typedef struct upir_map_s *upir_map;
typedef struct upir_spmd_s *upir_spmd;
typedef struct upir_event_s *upir_event;
typedef struct upir_graph_s *upir_graph;

/* ---- lifecycle ---------------------------------------------------------
 * world: NULL = one GPU, rank 0 of 1.  Otherwise rank/nranks of the
 * cluster-level SPMD (Fig. 1 target 'cluster'); nccl_id points at the
 * 128-byte ncclUniqueId produced on rank 0 by upir_comm_unique_id and
 * broadcast by the caller (e.g. torch.distributed).  compute_stream /
 * copy_stream: cudaStream_t values to run on, 0 = library-created streams.
 * nccl_id NULL with nranks > 1: a communicator-less world -- ranks exchange
 * data only through peer windows (upir_peer_*; fused world reductions, fused
 * halos, WORLD_BARRIER); NCCL-backed calls return UPIR_E_UNSUPPORTED.
 */
typedef struct {
    int32_t rank, nranks;
    const void *nccl_id;
    uintptr_t compute_stream, copy_stream;
} upir_world;

upir_status upir_init(int cuda_device, const upir_world *world, upir_ctx *out);
/* Waits for all work; UPIR_E_LEAK (and frees nothing) if maps are live. */
upir_status upir_finalize(upir_ctx ctx);
/* Produce a 128-byte NCCL unique id into out128 (rank 0, before upir_init). */
upir_status upir_comm_unique_id(void *out128);
/* The context's streams: which = 0 compute, 1 copy. */
upir_status upir_ctx_stream(upir_ctx ctx, int which, uintptr_t *out);
/* Counters since upir_init: out[0] H2D bytes enqueued by maps/updates,
 * out[1] D2H bytes, out[2] live maps, out[3] library kernels launched by this
 * context (a graph launch counts the kernels captured into the graph; a
 * capture itself launches nothing). */
upir_status upir_ctx_stats(upir_ctx ctx, int64_t out[4]);

/* ---- upir.data: mapping, movement, memory management (Figs. 5-6) -------
 * PAPER.md:782-808 data-mapping-property to | from | tofrom | allocate;
 * PAPER.md:843-854 data_movement / data_update (forward | backward) and
 * mm_allocator / mm_deallocator.
 *
 * Present table (reading c18): mapping a host pointer already present only
 * increments its refcount.  H2D copy (movement 'forward') on the 0 -> 1
 * transition for TO / TOFROM, D2H ('backward') on 1 -> 0 for FROM / TOFROM.
 * ALLOC and FROM get device memory without a copy.  Copies run on the copy
 * stream from pinned memory (host buffers are registered with
 * cudaHostRegister unless already pinned); the compute stream waits on them.
 * The host buffer must stay valid and unmodified until the next upir_sync.
 */
typedef enum { UPIR_MAP_TO = 1, UPIR_MAP_FROM = 2, UPIR_MAP_TOFROM = 3, UPIR_MAP_ALLOC = 4 } upir_map_kind;

/* Fig. 5 data-distribution pattern(block) across the ranks of a cluster
 * SPMD.  The global array has n_rows rows of row_elems elements of
 * elem_bytes each (a 1-D array: row_elems = 1).  Rank r owns the rows of the
 * static block rule over ranks (reading c20: q = n_rows / nranks, first
 * n_rows % nranks ranks get one more) plus halo_rows neighbour rows on each
 * side (clipped at the array ends).  The host pointer given to
 * upir_data_map is the GLOBAL host array; only the local rows move. */
typedef enum { UPIR_PATTERN_NONE = 0, UPIR_PATTERN_BLOCK = 1 } upir_pattern;
typedef struct {
    int32_t pattern;      /* upir_pattern */
    int32_t halo_rows;    /* >= 0 */
    int64_t n_rows;
    int64_t row_elems;
    int64_t elem_bytes;
} upir_dist;

upir_status upir_data_map(upir_ctx ctx, void *host, size_t bytes, upir_map_kind kind,
                          const upir_dist *dist /* NULL = whole array */, upir_map *out);
/* Register an existing device buffer (e.g. a torch tensor).  The caller keeps
 * ownership; unmap never frees it and never copies. */
upir_status upir_data_adopt(upir_ctx ctx, void *dev_ptr, size_t bytes,
                            const upir_dist *dist, upir_map *out);
/* Map exit: refcount - 1; at 0 the D2H copy (FROM/TOFROM) is enqueued after
 * all compute work so far, then the device memory is released. */
upir_status upir_data_unmap(upir_ctx ctx, upir_map map);
/* data_update: direction 0 = forward (host -> device), 1 = backward. */
upir_status upir_data_update(upir_ctx ctx, upir_map map, int direction);
/* data_update of an array section (Fig. 5 data-section [lo:len], stride 1):
 * bytes [byte_offset, byte_offset + bytes) of the map's LOCAL buffer (and of
 * the matching host range).  A forward update makes only LATER compute work
 * wait for THIS copy, so a loop over section k overlaps the copy of section
 * k+1 (chunk-pipelined map: overlap of data movement and
 * computation). */
upir_status upir_data_update_section(upir_ctx ctx, upir_map map, int64_t byte_offset, int64_t bytes,
                                     int direction);
/* direction UPIR_UPDATE_FORWARD_ASYNC (2): a forward section update that is
 * NOT ordered after earlier compute work (OpenMP 'target update to(...)
 * nowait'; the async attribute of a data movement): the
 * caller asserts that no compute work enqueued earlier touches the section.
 * Section copies then run back to back on the copy stream while the loop over
 * section k executes behind copy k only (chunk-pipelined map(to)). */
#define UPIR_UPDATE_FORWARD_ASYNC 2
/* Device pointer of the local buffer, the number of local elements (rows *
 * row_elems, halo included) and the global element index of its first
 * element. */
upir_status upir_data_device_ptr(upir_map map, void **dptr, int64_t *local_elems,
                                 int64_t *global_offset);
/* Block rule of upir_dist for rank r of nranks: owned rows [lo, hi).
 * Host-only; needs no device. */
upir_status upir_dist_owned_rows(int64_t n_rows, int32_t rank, int32_t nranks,
                                 int64_t *lo, int64_t *hi);

/* Halo plan of a BLOCK distribution (Fig. 7 send/recv between rank-adjacent
 * slabs, reading c20): for rank r, rows (global indices, half-open) to send
 * to / receive from the rank above (r-1) and below (r+1):
 *   out[0..1] send_up [lo,hi)   out[2..3] recv_up [lo,hi)
 *   out[4..5] send_dn [lo,hi)   out[6..7] recv_dn [lo,hi)
 * Empty ranges are [0,0).  Host-only; upir_sync(HALO) moves exactly these. */
upir_status upir_halo_plan(int64_t n_rows, int32_t halo_rows, int32_t rank, int32_t nranks,
                           int64_t out[8]);

/* ---- peer windows: NVLink peer memory between ranks (CUDA IPC) ----------
 * One process per GPU; the NVSwitch lets every GPU load/store every other
 * GPU's memory.  upir_peer_export writes a UPIR_PEER_REC_BYTES record (a
 * CUDA-IPC handle plus layout facts) for
 *   map == NULL : the context's peer window (signal counters and reduction
 *                 slots written by the other ranks), or
 *   map != NULL : a BLOCK-distributed map's local buffer (its halo rows are
 *                 the neighbours' peer-store targets).  A library-allocated
 *                 buffer is moved to an exportable block on first export
 *                 (device pointers taken earlier go stale); an adopted
 *                 buffer must be a cudaMalloc allocation (e.g. torch).
 * The caller moves records between ranks (e.g. all_gather_object) and calls
 * upir_peer_import(ctx, map, r, rec) for rank r's record: windows of every
 * rank (enables UPIR_WORLD_REDUCE in-kernel and the peer WORLD_BARRIER), map
 * buffers of ranks r +- 1 only (enables the fused halo below).
 *
 * Fused halo (PAPER.md:889 send/recv between rank-adjacent slabs, fused with
 * the sweep that produces the rows): a CLUSTER JACOBI5 loop whose out map
 * has imported neighbour buffers stores its first / last owned output row
 * also into the neighbours' halo rows of THEIR out buffers, and its tiles
 * that touch halo / boundary rows wait in the kernel until both neighbours
 * finished their previous sweep.  upir_sync(HALO) on a map written by such a
 * sweep returns at once (the exchange already happened).  Peer-mode sweeps
 * are collective: every rank executes the same sequence.  Unmapping a
 * peer-attached map first waits for the neighbours' last sweep.
 * Errors: UPIR_E_INVALID (bad record / rank / layout), UPIR_E_CUDA (IPC). */
#define UPIR_PEER_REC_BYTES 256
upir_status upir_peer_export(upir_ctx ctx, upir_map map, void *rec);
upir_status upir_peer_import(upir_ctx ctx, upir_map map, int32_t peer_rank, const void *rec);

/* ---- upir.spmd (Fig. 1) -------------------------------------------------
 * teams x units = CUDA grid x block (Figs. 11-12): team = CTA,
 * unit = thread, flat unit id g = team * num_units + unit.
 * num_units in [1, 1024], num_teams in [1, 2^31 - 1].  target GPU = this
 * device; CLUSTER = the same region on every rank of the world (the
 * worksharing loop is first block-distributed over ranks, reading c20). */
enum { UPIR_TARGET_GPU = 1, UPIR_TARGET_CLUSTER = 2 };
typedef struct {
    int32_t num_teams;
    int32_t num_units;
    uint32_t target;
    uint32_t reserved;
} upir_spmd_desc;

upir_status upir_spmd_launch(upir_ctx ctx, const upir_spmd_desc *desc, upir_spmd *out);
/* Closes the region: the region's implicit end barrier is stream order. */
upir_status upir_spmd_end(upir_spmd spmd);

/* ---- upir.loop + upir.loop_parallel worksharing (Fig. 3) ----------------
 * Canonical loop levels d < collapse, each [lb, ub) with step != 0
 * (reading c1; negative steps count down from lb).  Collapsed levels are
 * linearised row-major.
 *
 * schedule (readings c3-c8):
 *   STATIC, chunk 0  : unit u owns [u*q + min(u,r), +q + (u<r)), q = T/p, r = T%p
 *   STATIC, chunk c  : chunk k = [k*c, min((k+1)*c, T)) -> unit k mod p
 *   DYNAMIC, chunk c : same chunk partition (default c = 1); chunks are claimed
 *                      at run time; each unit's chunks are increasing
 *   GUIDED, chunk c  : chunks cut in dispatch order, each max(ceil(remaining /
 *                      p), c) long (default c = 1), claimed at run time like
 *                      DYNAMIC (1-D loops; tiled nests: UPIR_E_UNSUPPORTED)
 *   RUNTIME, AUTO    : resolve to STATIC
 * distribute: TEAMS_UNITS: p = teams*units over flat g;
 *   TEAMS: p = teams, executed by unit 0 of each team (reading c6);
 *   UNITS: p = units, requires num_teams == 1 (reading c7).
 *
 * Tiled nests (collapse 2, tile[0..1] > 0; PAPER.md:622/666 tiling before
 * parallelisation; reading c24): tiles of tile[0] x tile[1] anchored at
 * induction value 0 of each level, tile index row-major; the tile loop is
 * scheduled over TEAMS with (policy, chunk); inside a tile the tile-box
 * positions (row-major) are scheduled over UNITS with (inner_policy,
 * inner_chunk); a box position outside [lb, ub) performs no iteration.
 */
typedef enum {
    UPIR_SCHED_STATIC = 0, UPIR_SCHED_DYNAMIC = 1, UPIR_SCHED_GUIDED = 2,
    UPIR_SCHED_RUNTIME = 3, UPIR_SCHED_AUTO = 4
} upir_sched;
typedef enum { UPIR_DIST_TEAMS = 1, UPIR_DIST_UNITS = 2, UPIR_DIST_TEAMS_UNITS = 3 } upir_distribute;

#define UPIR_NOWAIT 1u  /* no implicit end barrier: the host does not wait */
/* UPIR_TILE_COLMAJOR (tiled JACOBI5 nests; reading c35 of DESIGN.md): the
 * tile loop enumerates the tiles column-major -- tile id = (tj - tj0) * ntr +
 * (ti - ti0) -- instead of row-major (reading c24).  The paper's tiling
 * fixes no order; with schedule(static) a team then owns a
 * vertical run of tiles and re-reads its own previous tile's boundary row
 * from L2 instead of a row another team fetched.  Trace records index tiles
 * by this id.  Other bodies: UPIR_E_UNSUPPORTED. */
#define UPIR_TILE_COLMAJOR 4u
/* UPIR_TILE_REVERSE (tiled JACOBI5 nests; reading c38 of DESIGN.md): tile id
 * k enumerates the tile grid from its last tile -- id k is the tile the
 * plain order numbers ntiles - 1 - k (row- or column-major) -- with the
 * tile-loop schedule and the intra-tile rule unchanged; trace records index
 * tiles by this id.  Sweeps that alternate it start on the rows the previous
 * sweep wrote last (still in L2).  Other bodies: UPIR_E_UNSUPPORTED. */
#define UPIR_TILE_REVERSE 16u
/* UPIR_HALO_EXPLICIT (JACOBI5 on a CLUSTER target whose out map has imported
 * neighbour buffers): do not fuse the halo exchange into the sweep (no peer
 * stores of the boundary rows, no in-kernel neighbour waits); the program
 * exchanges with upir_sync(HALO), synchronously or async (arrive-compute /
 * JOIN), over the same peer mappings.  Without imported buffers: no effect.
 * Other bodies: ignored. */
#define UPIR_HALO_EXPLICIT 32u
/* UPIR_WORLD_REDUCE: the loop's reductions are combined over all ranks as part
 * of the loop (Fig. 7 'allreduce' with ranks as units fused into the loop's
 * end barrier): every rank receives
 *   init (+) P_0 (+) P_1 (+) ... (+) P_{N-1}   (ascending rank order)
 * where P_r is rank r's combination of its units' partials (int64, or fp64
 * for F32 rounded once; the original value counted once).  With every rank's
 * peer window imported the last team of each rank exchanges the partials
 * through NVLink peer memory inside the loop kernel; otherwise (communicator
 * only, or UPIR_WORLD_VIA_COMM) the loop's last team writes P_r to a context
 * scratch word pair, an ncclAllGather collects them and one combine kernel
 * applies init in ascending rank order -- the same arithmetic, so both paths
 * give identical bits.  Collective: every rank must execute the loop.
 * nranks == 1: no effect. */
#define UPIR_WORLD_REDUCE 2u
/* UPIR_WORLD_VIA_COMM: with UPIR_WORLD_REDUCE, combine over ranks through the
 * communicator (NCCL all-gather) even when the peer windows are imported
 * (measurement of the NCCL path next to the fused one).  At nranks == 1 the
 * same partial / gather / combine sequence runs with a device copy as the
 * gather (the result equals the plain loop's). */
#define UPIR_WORLD_VIA_COMM 8u

typedef struct {
    int32_t collapse;        /* 1..2 */
    int32_t policy;          /* upir_sched */
    int64_t lb[3], ub[3], step[3];
    int64_t tile[3];         /* 0 = untiled */
    int64_t chunk;           /* 0 = unspecified */
    int32_t distribute;      /* upir_distribute */
    int32_t inner_policy;    /* upir_sched, tiled nests only */
    int64_t inner_chunk;
    uint32_t flags;
    uint32_t simdlen;        /* loop_parallel simd(simdlen); 0 or 1 = none (see below) */
} upir_loop_desc;
/* simd(simdlen(s)) with worksharing (reading c33):
 * the loop the units execute is strip-mined into SIMD groups of s
 * consecutive iterations (the last one ragged) and the schedule distributes
 * whole groups -- chunk c becomes s*ceil(c/s) (OpenMP's simd schedule
 * modifier; dynamic / guided default: one group), static without chunk is
 * the block rule over ceil(T/s) groups, CLUSTER loops split groups over
 * ranks -- and a unit executes each group as one s-lane vector.  Applies to
 * the 1-D loops (AXPY, REDUCE, MATVEC rows), to the intra-tile position loop
 * of tiled nests (JACOBI5, STENCIL2D: inner_chunk becomes s*ceil(c/s)) and to
 * MATVEC's k-loop under distribute(teams); MATMUL's intra-tile work is a
 * tensor-core operation already (no observable effect).  s <= 4096. */

/* Loop bodies (the kernels of the paper's evaluation):
 *  AXPY    : y[i] = y[i] + alpha * x[i]    (Figs. 9/11)
 *            in0 = x, out = y (fp32).  Reductions (optional) combine y'[i].
 *  REDUCE  : reductions combine in0[i] (int64 or fp32).
 *  JACOBI5 : out[i][j] = 0.25*((in[i-1][j] + in[i+1][j]) + (in[i][j-1] +
 *            in[i][j+1])) over the loop's (i, j) space (collapse 2); in0 = in,
 *            out = out, fp32, row pitch ld[0] elements, dims[0] = n rows.
 *  MATMUL  : C[i][j] = sum_k A[i][k] * B[k][j] over the loop's (i, j) space
 *            (collapse 2, k sequential inside the iteration); in0 = A (M x K),
 *            in1 = B (K x N), out = C (M x N fp32), row-major; dims = (K, M,
 *            N), ld = (lda, ldb, ldc) in elements (multiples of 8).  dtype
 *            BF16: bf16 inputs, fp32 accumulation on tcgen05 tensor cores;
 *            F32: fp32 inputs via 3xTF32 (kind::tf32, D += lo_a*hi_b +
 *            hi_a*lo_b + hi_a*hi_b; A and B are split into tf32 hi / lo
 *            copies in HBM by one elementwise pass before the loop kernel).
 *            Team geometry (the tile loop runs over the teams, reading c24):
 *              BF16, 256 units: one CTA per team, 128 x 256 tiles;
 *              BF16, 512 units: a team is a 2-CTA cluster (CTA pair,
 *                tcgen05.mma.cta_group::2), 256 x 256 tiles;
 *              F32, 384 units: one CTA per team, 128 x 256 tiles;
 *              F32, 768 units: CTA pair, 256 x 256 tiles.
 *            Other unit counts are rejected (UPIR_E_INVALID), never clamped.
 *  MATVEC  : y[i] = sum_k A[i][k] * x[k] over the loop's rows i (collapse 1,
 *            step 1, the paper's fourth kernel); in0 = A (M x K
 *            fp32, row pitch ld[0]), in1 = x (K), out = y (M); dims = (K, M).
 *            distribute(teams): rows over teams, the k-loop over the team's
 *            units with schedule(static, inner_chunk, default 4) and a
 *            reduction(+); distribute(teams,units) / (units): rows over the
 *            flat units, k sequential per unit.
 *  STENCIL2D: out[i][j] = sum_{a,b in [-R,R]} w[a+R][b+R] * in[i+a][j+b]
 *            (the paper's "2D stencil, filter size = 7"; the
 *            weights are an input, reading c28); in0 = in, in1 = w (F x F
 *            fp32, F = 2R+1 in {3,5,7}), out = out; ld[0] = row pitch,
 *            dims = (ny, F).  Tiled like JACOBI5 (tiles BM x BN in {16x128,
 *            8x64, 16x512, 16x1024, 8x512, 8x1024, 8x256, 4x512, 4x256}).
 * The element index used by a body is the induction value itself (global
 * index; for distributed maps the runtime subtracts the local offset). */
typedef enum { UPIR_BODY_AXPY = 0, UPIR_BODY_REDUCE = 1, UPIR_BODY_JACOBI5 = 2,
               UPIR_BODY_MATMUL = 3, UPIR_BODY_MATVEC = 4, UPIR_BODY_STENCIL2D = 5 } upir_body_kind;
typedef struct {
    int32_t kind;            /* upir_body_kind */
    int32_t dtype;           /* element type of in0 (matmul: of A and B) */
    upir_map in0, in1, out;
    double alpha;
    int64_t ld[3];
    int64_t dims[3];
} upir_body;

/* upir.sync reduction ([REM] 929-948 mode all-unit).
 * Private copies start at the identity (sum 0, max -inf / INT64_MIN, min
 * +inf / INT64_MAX, reading c9); result = init (+) all partials.  init: host
 * pointer to one element of dtype (NULL = identity).  dev_result: device
 * pointer to one element of dtype; valid after the next upir_sync (or in
 * stream order).  Combining order is a fixed tree (warp butterfly, team,
 * ascending team slots) -- bit-reproducible for a fixed geometry (c10). */
typedef enum { UPIR_OP_SUM = 0, UPIR_OP_MAX = 1, UPIR_OP_MIN = 2 } upir_op;
typedef struct {
    int32_t op;              /* upir_op */
    int32_t dtype;           /* UPIR_I64 | UPIR_F32 */
    const void *init;
    void *dev_result;
} upir_reduction;

/* Execute the loop on the region.  reds: 0..2 reductions over the same loop
 * (NULL if n_reds == 0).  trace: NULL or an int32 map of 3*T elements
 * [team[T], unit[T], hits[T]] (hits pre-zeroed by the caller) -- every
 * executed iteration t records the (team, unit) that ran it and increments
 * hits[t] (the same kernel as the untraced body, compiled with tracing).
 * For tiled nests t is the box position index tile*tile_elems + pos and the
 * recorded unit is the intra-tile unit. */
upir_status upir_loop_exec(upir_spmd spmd, const upir_loop_desc *loop, const upir_body *body,
                           const upir_reduction *reds, int32_t n_reds, upir_map trace);

/* Host-only helpers (no device needed): normalised trip counts of a loop
 * descriptor, T = prod T_d over collapsed levels. */
upir_status upir_loop_normalize(const upir_loop_desc *loop, int64_t *T_total, int64_t T_d[3]);
/* Full validation of (spmd, loop, body kind, reductions) without a context. */
upir_status upir_loop_validate(const upir_spmd_desc *spmd, const upir_loop_desc *loop,
                               int32_t body_kind, const upir_reduction *reds, int32_t n_reds);
/* The schedule's chunks for unit u (host mirror of the device engine, for
 * tests): writes up to cap chunks, *count = total owned.  DYNAMIC returns
 * UPIR_E_INVALID (its assignment is decided at run time). */
upir_status upir_schedule_chunks(int32_t policy, int64_t chunk, int64_t T, int64_t p, int64_t u,
                                 int64_t *lo, int64_t *hi, int64_t cap, int64_t *count);

/* ---- upir.sync (Fig. 7) -------------------------------------------------
 * upir_reduce: standalone reduction / allreduce.
 *   DEVICE : dev_out[0] = (+) over the count elements of dev_in (fixed tree).
 *   WORLD  : 'allreduce' with ranks as primary/secondary units: dev_in holds
 *            count elements on every rank; every rank receives, element-wise,
 *            the combination over ranks in ascending rank order (fp32 in fp64,
 *            rounded once: deterministic and identical on every rank, reading
 *            c10).  Transport: with every rank's peer window imported and
 *            count <= 65536, one kernel stages dev_in in this rank's window,
 *            publishes it to every rank and combines all ranks' staged values
 *            over NVLink; otherwise NCCL all-gather + the same ordered
 *            combine (a communicator-less world: UPIR_E_UNSUPPORTED). */
typedef enum { UPIR_SCOPE_DEVICE = 0, UPIR_SCOPE_WORLD = 1 } upir_scope;
upir_status upir_reduce(upir_ctx ctx, int32_t op, int32_t dtype, const void *dev_in,
                        int64_t count, void *dev_out, int32_t scope);
/* upir_reduce_async: the WORLD allreduce as the async two-step sync
 * (PAPER.md:880-882 'arrive-compute' / 'wait-release'; SURVEY 8(f) NEXT #1
 * 'async allreduce'): the all-gather and the ordered combine are enqueued on
 * the copy stream after the compute work issued so far (they read dev_in as
 * that work left it), into a stream-ordered scratch of their own; compute
 * work issued afterwards does NOT wait for them.  *token (NULL on entry)
 * receives their completion: upir_sync(JOIN, token) makes later compute work
 * wait (device-side), upir_sync(WAIT, token) blocks the host.  dev_in must
 * not be overwritten before the token is released; until then this rank
 * issues no other WORLD reduction.  nranks == 1: a device copy replaces the
 * all-gather.  Transport as upir_reduce(WORLD).  Errors as upir_reduce; a non-empty *token is
 * UPIR_E_INVALID. */
upir_status upir_reduce_async(upir_ctx ctx, int32_t op, int32_t dtype, const void *dev_in,
                              int64_t count, void *dev_out, upir_event *token);

/* upir_sync kinds:
 *   BARRIER       : host waits for all work of this context; reports sticky
 *                   asynchronous errors (the implicit barrier).
 *   WORLD_BARRIER : BARRIER on every rank, then a device-side barrier over
 *                   ranks (Fig. 7 barrier with rank units).
 *   ARRIVE        : async two-step, step 'arrive-compute':
 *                   records a token after the work enqueued so far; *token out.
 *   WAIT          : step 'wait-release': the host waits for *token and frees it.
 *   HALO          : send/recv of halo rows of a BLOCK-distributed map with
 *                   ranks r-1 / r+1 (Fig. 7 send/recv), in stream order.
 *                   Transport: when the map has its neighbours' buffers
 *                   imported (upir_peer_import) and every rank's peer window
 *                   is imported, one kernel stores this rank's boundary rows
 *                   into the neighbours' halo rows over the peer mappings
 *                   (NVLink) and waits for theirs (release / acquire
 *                   counters in the peer windows, shared with the fused
 *                   sweeps' protocol); otherwise NCCL send/recv (a
 *                   communicator-less world: UPIR_E_UNSUPPORTED).  A map
 *                   last written by a fused peer-mode sweep is already
 *                   exchanged: HALO then only waits (stream order) for the
 *                   neighbours' deliveries of that sweep.  Both share one generation counter per
 *                   rank: a fused sweep may not run while an async exchange
 *                   of this rank is still in flight (JOIN first).
 *                   With token != NULL (*token == NULL on entry) it is the
 *                   async 'arrive-compute' step: the exchange runs on the copy
 *                   stream, overlapping later compute work, and *token
 *                   receives its completion event.
 *   JOIN          : async 'wait-release' on the DEVICE: later compute work
 *                   waits for *token (no host block); the token is freed.
 *                   UPIR_E_SYNC without a token. */
typedef enum { UPIR_SYNC_BARRIER = 0, UPIR_SYNC_WORLD_BARRIER = 1, UPIR_SYNC_ARRIVE = 2,
               UPIR_SYNC_WAIT = 3, UPIR_SYNC_HALO = 4, UPIR_SYNC_JOIN = 5 } upir_sync_kind;
upir_status upir_sync(upir_ctx ctx, int32_t kind, upir_map halo_map, upir_event *token);

/* ---- CUDA-graph capture of a loop sequence (e.g. 100 Jacobi sweeps) ------ */
upir_status upir_graph_begin(upir_ctx ctx);
upir_status upir_graph_end(upir_ctx ctx, upir_graph *out);
upir_status upir_graph_launch(upir_ctx ctx, upir_graph graph);
upir_status upir_graph_destroy(upir_graph graph);

/* ---- synthetic inputs on the device (counter-based splitmix64) -----------
 * The recipe of DESIGN.md "Input recipe", implemented independently of the
 * host generator (synth/).  Fills the local buffer of map m: element e gets
 * the value of global index global_offset_of(m) + e + index_base.
 * dist: 0 = f32 U[0,1), 1 = f32 U[-1,1), 2 = i64 U[-2^28, 2^28),
 *       3 = bf16 U[-1,1), 4 = Jacobi initial grid (f32; n_cols = row length,
 *       n_rows = global rows: interior U[0,1), top row 1, other boundary 0). */
upir_status upir_synth_fill(upir_ctx ctx, upir_map m, int32_t dist, uint64_t stream,
                            int64_t index_base, int64_t n_rows, int64_t n_cols);

#ifdef __cplusplus
}
#endif
#endif /* UPIR_H */
