/*
 * upir_oracle.c -- plain, slow, sequential CPU oracle of the UPIR
 * data-parallel loop path (arXiv 2209.10643).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * It shares no code, header, table or helper with the CUDA path
 * (paper_2209_10643_b200/, include/upir.h): its descriptor encoding below is
 * its own.  Floating point is evaluated in fp64, integers exactly in int64
 * (two's-complement wrap via uint64, reading c12 of DESIGN.md).
 *
 * What it interprets (Fig. 3 "upir.loop" /
 * "upir.loop_parallel worksharing"; SPEC.md:397-426 interpreter):
 *     for u in 0..p-1 (ascending)
 *       for chunk in schedule(u) (ascending)
 *         for t in chunk: body(t), accumulating partial[u]
 *     result = init (+) partial[0] (+) ... (+) partial[p-1]
 * Where the method reaches a plain result exactly (axpy, Jacobi, matmul:
 * every output element is produced by exactly one iteration) the oracle
 * computes that plain definition directly.
 *
 * Readings: c1 half-open bounds,
 * c3 default static, c4 static remainder to low ids, c5 flat
 * p = teams*units, c8 dynamic dispatcher, c9 identities, c10 combine order,
 * c12 integer wrap, c13 fmax semantics, c16 Jacobi definition, c17 matmul.
 *
 * Parity pins: every function here is pinned by tests/test_oracle_*.py
 * against something other than itself (SPEC worked examples, libgomp,
 * closed forms, invariants, brute force, numpy float64 matmul).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ---- oracle-private descriptor encoding ------------------------------- */
enum { ORC_STATIC = 0, ORC_DYNAMIC = 1, ORC_GUIDED = 2, ORC_RUNTIME = 3, ORC_AUTO = 4 };
enum { ORC_SUM = 0, ORC_MAX = 1, ORC_MIN = 2 };

/* o1. Trip count of one canonical loop level (Fig. 3
 * induction/lowerBound/upperBound/step; half-open reading c1).
 *   T = max(0, ceil((ub - lb) / step))   for step > 0
 *   T = max(0, ceil((lb - ub) / -step))  for step < 0 (normalised)
 * step == 0 is invalid: returns -1. */
int64_t orc_trip_count(int64_t lb, int64_t ub, int64_t step)
{
    if (step == 0) return -1;
    if (step > 0) {
        if (ub <= lb) return 0;
        return (ub - lb + step - 1) / step;
    }
    if (lb <= ub) return 0;
    return (lb - ub + (-step) - 1) / (-step);
}

/* o1 collapse.  Row-major (lexicographic) de-linearisation of the collapsed
 * index t in [0, prod T_d) into per-level normalised indices k_d
 * ("collapse"; i = t / T_j, j = t % T_j). */
void orc_delinearize(int collapse, const int64_t *T, int64_t t, int64_t *k)
{
    for (int d = collapse - 1; d >= 0; --d) {
        k[d] = t % T[d];
        t /= T[d];
    }
}

/* ---- o2/o3: the worksharing schedule ---------------------------------- */
/* Number of chunks of size c covering [0,T). */
static int64_t n_chunks(int64_t T, int64_t c) { return (T + c - 1) / c; }

/* Chunks owned by unit u under (policy, chunk) over T iterations and p
 * units.  Writes up to cap chunks [lo,hi) in execution order and returns the
 * total number owned (which may exceed cap).
 *
 * static, no chunk (reading c4):
 *     q = T / p, r = T % p; unit u owns [u*q + min(u,r), +q + (u<r)).
 * static, chunk c: chunk k = [k*c, min((k+1)*c, T)) goes to unit k mod p.
 * dynamic, chunk c (default 1): same chunk partition; chunk k is handed by
 *     the deterministic dispatcher (reading c8): units wait in a
 *     FIFO queue initially ordered by id; the unit at the head takes the next
 *     chunk, runs it, and re-enters the queue at the tail.
 * runtime / auto resolve to static (reading c3).
 * guided, chunk c (default 1; PAPER.md:644 'guided'): chunks
 *     are cut in dispatch order, each max(ceil(remaining / p), c) long
 *     (clipped at T), remaining = T - start of the chunk; handed out by the
 *     same deterministic dispatcher as dynamic. */
int64_t orc_schedule_chunks(int policy, int64_t chunk, int64_t T, int64_t p,
                            int64_t u, int64_t *lo, int64_t *hi, int64_t cap)
{
    int64_t cnt = 0;
    if (p <= 0 || u < 0 || u >= p || T < 0) return -1;
    if (policy == ORC_RUNTIME || policy == ORC_AUTO) { policy = ORC_STATIC; chunk = 0; }
    if (policy == ORC_GUIDED) {
        int64_t c = chunk <= 0 ? 1 : chunk;
        int64_t *queue = (int64_t *)malloc(sizeof(int64_t) * (size_t)p);
        if (!queue) return -1;
        int64_t head = 0, count = p, start = 0;
        for (int64_t i = 0; i < p; ++i) queue[i] = i;
        while (start < T) {
            int64_t rem = T - start;
            int64_t len = (rem + p - 1) / p;          /* ceil(remaining / p) */
            if (len < c) len = c;
            if (len > rem) len = rem;
            int64_t w = queue[head];
            head = (head + 1) % p; --count;
            if (w == u) {
                if (cnt < cap) { lo[cnt] = start; hi[cnt] = start + len; }
                ++cnt;
            }
            queue[(head + count) % p] = w; ++count;
            start += len;
        }
        free(queue);
        return cnt;
    }
    if (policy == ORC_STATIC && chunk <= 0) {
        int64_t q = T / p, r = T % p;
        int64_t start = u * q + (u < r ? u : r);
        int64_t len = q + (u < r ? 1 : 0);
        if (len > 0) {
            if (cap > 0) { lo[0] = start; hi[0] = start + len; }
            cnt = 1;
        }
        return cnt;
    }
    if (policy == ORC_STATIC) {
        int64_t nc = n_chunks(T, chunk);
        for (int64_t k = u; k < nc; k += p) {
            if (cnt < cap) { lo[cnt] = k * chunk; hi[cnt] = (k + 1) * chunk < T ? (k + 1) * chunk : T; }
            ++cnt;
        }
        return cnt;
    }
    if (policy == ORC_DYNAMIC) {
        int64_t c = chunk <= 0 ? 1 : chunk;
        int64_t nc = n_chunks(T, c);
        /* the dispatcher: a FIFO of waiting unit ids */
        int64_t *queue = (int64_t *)malloc(sizeof(int64_t) * (size_t)p);
        if (!queue) return -1;
        int64_t head = 0, count = p;
        for (int64_t i = 0; i < p; ++i) queue[i] = i;
        for (int64_t k = 0; k < nc; ++k) {
            int64_t w = queue[head];               /* unit at the head */
            head = (head + 1) % p; --count;
            if (w == u) {
                if (cnt < cap) { lo[cnt] = k * c; hi[cnt] = (k + 1) * c < T ? (k + 1) * c : T; }
                ++cnt;
            }
            queue[(head + count) % p] = w; ++count; /* back to the tail */
        }
        free(queue);
        return cnt;
    }
    return -1;
}

/* loop_parallel simd(simdlen(s)) combined with worksharing (PAPER.md:638,
 * 647-648 'simd' / 'simdlen'; reading c33): the loop is strip-mined into
 * ceil(T/s) SIMD groups of s consecutive iterations (the last one ragged),
 * the worksharing schedule distributes the GROUPS (a chunk of c iterations
 * becomes ceil(c/s) groups -- OpenMP's simd schedule modifier, chunk
 * s*ceil(c/s)), and a unit executes each group as one s-lane vector.  The
 * chunks below are the expansion of the group chunks back to iterations. */
int64_t orc_schedule_chunks_simd(int policy, int64_t chunk, int64_t simdlen, int64_t T, int64_t p,
                                 int64_t u, int64_t *lo, int64_t *hi, int64_t cap)
{
    if (simdlen <= 1) return orc_schedule_chunks(policy, chunk, T, p, u, lo, hi, cap);
    if (T < 0) return -1;
    int64_t s = simdlen;
    int64_t Tg = (T + s - 1) / s;
    int64_t cg = chunk <= 0 ? chunk : (chunk + s - 1) / s;
    int64_t n = orc_schedule_chunks(policy, cg, Tg, p, u, lo, hi, cap);
    for (int64_t k = 0; k < n && k < cap; ++k) {
        lo[k] = lo[k] * s;
        hi[k] = hi[k] * s < T ? hi[k] * s : T;
    }
    return n;
}

/* Executor of every normalised iteration t in [0,T): owner[t] = unit id in
 * [0,p), obtained by running the interpreter loop nest of the schedule
 * (for u ascending, for chunk of u, for t in chunk).  Returns 0, or -1. */
int orc_owner_map_simd(int policy, int64_t chunk, int64_t simdlen, int64_t T, int64_t p, int64_t *owner);
int orc_owner_map(int policy, int64_t chunk, int64_t T, int64_t p, int64_t *owner)
{
    return orc_owner_map_simd(policy, chunk, 1, T, p, owner);
}

int orc_owner_map_simd(int policy, int64_t chunk, int64_t simdlen, int64_t T, int64_t p, int64_t *owner)
{
    int64_t cap = 1 << 16;
    int64_t *lo = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
    int64_t *hi = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
    if (!lo || !hi) { free(lo); free(hi); return -1; }
    for (int64_t t = 0; t < T; ++t) owner[t] = -1;
    for (int64_t u = 0; u < p; ++u) {
        int64_t n = orc_schedule_chunks_simd(policy, chunk, simdlen, T, p, u, lo, hi, cap);
        if (n < 0) { free(lo); free(hi); return -1; }
        if (n > cap) {  /* grow and redo */
            free(lo); free(hi); cap = n;
            lo = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
            hi = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
            if (!lo || !hi) { free(lo); free(hi); return -1; }
            n = orc_schedule_chunks_simd(policy, chunk, simdlen, T, p, u, lo, hi, cap);
        }
        for (int64_t c = 0; c < n; ++c)
            for (int64_t t = lo[c]; t < hi[c]; ++t) {
                if (owner[t] != -1) { free(lo); free(hi); return -2; } /* overlap */
                owner[t] = u;
            }
    }
    free(lo); free(hi);
    return 0;
}

/* ---- o4: axpy body (Fig. 9, 1180-1186 Fig. 11) ------
 *   y[i] = y[i] + a * x[i]   for every iteration i = lb + k*step, k in [0,T)
 * evaluated in fp64 from the fp32 inputs (reading c14: a is real-valued).
 * Each iteration writes its own element, so the schedule only partitions:
 * the oracle evaluates the plain definition.  y_out receives all n elements
 * (untouched ones copied from y). */
int orc_axpy(int64_t n, int64_t lb, int64_t ub, int64_t step, double a,
             const float *x, const float *y, double *y_out)
{
    int64_t T = orc_trip_count(lb, ub, step);
    if (T < 0) return -1;
    for (int64_t i = 0; i < n; ++i) y_out[i] = (double)y[i];
    for (int64_t k = 0; k < T; ++k) {
        int64_t i = lb + k * step;
        if (i < 0 || i >= n) return -2;
        y_out[i] = (double)y[i] + a * (double)x[i];
    }
    return 0;
}

/* ---- o5: reductions (Fig. 7 sync 'reduction'; [REM]
 * 929-948 reduction-mode all-unit; SPEC.md:400/424 ascending unit order).
 * Private copies start at the identity (reading c9); unit u accumulates over
 * its chunks in execution order; partials combine with init in ascending
 * unit id. */
static uint64_t i64_combine(int op, uint64_t acc, int64_t v)
{
    if (op == ORC_SUM) return acc + (uint64_t)v;             /* wraps (c12) */
    if (op == ORC_MAX) return ((int64_t)acc > v) ? acc : (uint64_t)v;
    return ((int64_t)acc < v) ? acc : (uint64_t)v;
}

static uint64_t i64_identity(int op)
{
    if (op == ORC_SUM) return 0;
    if (op == ORC_MAX) return (uint64_t)INT64_MIN;
    return (uint64_t)INT64_MAX;
}

/* x is indexed by the induction value i = lb + k*step.  partials (may be
 * NULL) receives the p private results.  Returns 0 and writes *result, or a
 * negative error. */
int orc_reduce_i64(int op, int64_t n, int64_t lb, int64_t ub, int64_t step,
                   int policy, int64_t chunk, int64_t p, const int64_t *x,
                   int64_t init, int64_t *partials, int64_t *result)
{
    int64_t T = orc_trip_count(lb, ub, step);
    if (T < 0 || p <= 0) return -1;
    int64_t cap = 1;
    int64_t *lo = (int64_t *)malloc(sizeof(int64_t));
    int64_t *hi = (int64_t *)malloc(sizeof(int64_t));
    uint64_t total = (uint64_t)init;
    for (int64_t u = 0; u < p; ++u) {
        int64_t nc = orc_schedule_chunks(policy, chunk, T, p, u, lo, hi, cap);
        if (nc < 0) { free(lo); free(hi); return -1; }
        if (nc > cap) {
            free(lo); free(hi); cap = nc;
            lo = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
            hi = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
            nc = orc_schedule_chunks(policy, chunk, T, p, u, lo, hi, cap);
        }
        uint64_t part = i64_identity(op);
        for (int64_t c = 0; c < nc; ++c)
            for (int64_t k = lo[c]; k < hi[c]; ++k) {
                int64_t i = lb + k * step;
                if (i < 0 || i >= n) { free(lo); free(hi); return -2; }
                part = i64_combine(op, part, x[i]);
            }
        if (partials) partials[u] = (int64_t)part;
        total = i64_combine(op, total, (int64_t)part);
    }
    free(lo); free(hi);
    *result = (int64_t)total;
    return 0;
}

/* fp32 data, fp64 evaluation.  max/min follow fmax/fmin (reading c13). */
static double f_identity(int op)
{
    if (op == ORC_SUM) return 0.0;
    if (op == ORC_MAX) return -INFINITY;
    return INFINITY;
}

static double f_combine(int op, double acc, double v)
{
    if (op == ORC_SUM) return acc + v;
    if (op == ORC_MAX) return fmax(acc, v);
    return fmin(acc, v);
}

int orc_reduce_f32(int op, int64_t n, int64_t lb, int64_t ub, int64_t step,
                   int policy, int64_t chunk, int64_t p, const float *x,
                   double init, double *partials, double *result)
{
    int64_t T = orc_trip_count(lb, ub, step);
    if (T < 0 || p <= 0) return -1;
    int64_t cap = 1;
    int64_t *lo = (int64_t *)malloc(sizeof(int64_t));
    int64_t *hi = (int64_t *)malloc(sizeof(int64_t));
    double total = init;
    for (int64_t u = 0; u < p; ++u) {
        int64_t nc = orc_schedule_chunks(policy, chunk, T, p, u, lo, hi, cap);
        if (nc < 0) { free(lo); free(hi); return -1; }
        if (nc > cap) {
            free(lo); free(hi); cap = nc;
            lo = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
            hi = (int64_t *)malloc(sizeof(int64_t) * (size_t)cap);
            nc = orc_schedule_chunks(policy, chunk, T, p, u, lo, hi, cap);
        }
        double part = f_identity(op);
        for (int64_t c = 0; c < nc; ++c)
            for (int64_t k = lo[c]; k < hi[c]; ++k) {
                int64_t i = lb + k * step;
                if (i < 0 || i >= n) { free(lo); free(hi); return -2; }
                part = f_combine(op, part, (double)x[i]);
            }
        if (partials) partials[u] = part;
        total = f_combine(op, total, part);
    }
    free(lo); free(hi);
    *result = total;
    return 0;
}

/* ---- o6: Jacobi 5-point (north_star; reading c16, c25) ----------------
 * One sweep: out[i][j] = 0.25*((in[i-1][j] + in[i+1][j]) + (in[i][j-1] +
 * in[i][j+1])) for 1 <= i < ny-1, 1 <= j < nx-1; boundary copied unchanged.
 * S sweeps ping-pong between two grids, evaluated in fp64 from the fp32
 * initial grid.  out receives the grid after S sweeps. */
int orc_jacobi5(int64_t ny, int64_t nx, int64_t S, const float *init, double *out)
{
    if (ny < 1 || nx < 1 || S < 0) return -1;
    size_t N = (size_t)ny * (size_t)nx;
    double *a = (double *)malloc(N * sizeof(double));
    double *b = (double *)malloc(N * sizeof(double));
    if (!a || !b) { free(a); free(b); return -1; }
    for (size_t e = 0; e < N; ++e) a[e] = (double)init[e];
    memcpy(b, a, N * sizeof(double));
    for (int64_t s = 0; s < S; ++s) {
        for (int64_t i = 1; i < ny - 1; ++i)
            for (int64_t j = 1; j < nx - 1; ++j)
                b[i * nx + j] = 0.25 * ((a[(i - 1) * nx + j] + a[(i + 1) * nx + j]) +
                                        (a[i * nx + j - 1] + a[i * nx + j + 1]));
        double *t = a; a = b; b = t;
    }
    memcpy(out, a, N * sizeof(double));
    free(a); free(b);
    return 0;
}

/* Light-cone window of the same computation, for parity at full size.
 * win holds the fp32 initial values of global rows [wr0, wr0+wy) and columns
 * [wc0, wc0+wx) of an ny x nx grid.  After S sweeps the value of a point is a
 * function of the initial values within Manhattan distance S (the 5-point
 * light cone), so points at row and column distance >= S from every window
 * edge that is NOT a global boundary are exact. The window is swept S times (interior points of the
 * global grid that are also strictly inside the window are updated; window
 * edge points keep their initial values -- wrong after one sweep, but the
 * error front advances one point per sweep).  out (wy*wx doubles) receives
 * the swept window; the caller reads only the exact core. */
int orc_jacobi5_window(int64_t ny, int64_t nx, int64_t S, int64_t wr0, int64_t wc0,
                       int64_t wy, int64_t wx, const float *win, double *out)
{
    if (wy < 1 || wx < 1 || S < 0) return -1;
    size_t N = (size_t)wy * (size_t)wx;
    double *a = (double *)malloc(N * sizeof(double));
    double *b = (double *)malloc(N * sizeof(double));
    if (!a || !b) { free(a); free(b); return -1; }
    for (size_t e = 0; e < N; ++e) a[e] = (double)win[e];
    memcpy(b, a, N * sizeof(double));
    for (int64_t s = 0; s < S; ++s) {
        for (int64_t li = 1; li < wy - 1; ++li) {
            int64_t gi = wr0 + li;
            if (gi < 1 || gi >= ny - 1) continue;
            for (int64_t lj = 1; lj < wx - 1; ++lj) {
                int64_t gj = wc0 + lj;
                if (gj < 1 || gj >= nx - 1) continue;
                b[li * wx + lj] = 0.25 * ((a[(li - 1) * wx + lj] + a[(li + 1) * wx + lj]) +
                                          (a[li * wx + lj - 1] + a[li * wx + lj + 1]));
            }
        }
        double *t = a; a = b; b = t;
    }
    memcpy(out, a, N * sizeof(double));
    free(a); free(b);
    return 0;
}

/* ---- o7: matmul (north_star; reading c17) ---------------
 * C[i][j] = sum_k A[i][k] * B[k][j], row-major, fp64 from the exact input
 * values (bf16 inputs are passed as their exact fp32 values).  Only the rows
 * listed in `rows` (nrows of them) are computed, into C[r][*] of a
 * nrows x N output, so full-size parity can sample rows. */
int orc_matmul_rows(int64_t M, int64_t N, int64_t K, const float *A, const float *B,
                    const int64_t *rows, int64_t nrows, double *C)
{
    for (int64_t r = 0; r < nrows; ++r) {
        int64_t i = rows[r];
        if (i < 0 || i >= M) return -2;
        for (int64_t j = 0; j < N; ++j) {
            double acc = 0.0;
            for (int64_t k = 0; k < K; ++k)
                acc += (double)A[i * K + k] * (double)B[k * N + j];
            C[r * N + j] = acc;
        }
    }
    return 0;
}

/* Tile -> team owner map of a tiled collapse(2) nest (reading c24): the
 * iteration space [0,R) x [0,Cn) is cut into tiles of tm x tn (row-major tile
 * order, ragged last tiles); the tile loop is scheduled over p teams with
 * (policy, chunk).  owner[tile] = team id. */
int orc_tile_owner(int64_t R, int64_t Cn, int64_t tm, int64_t tn, int policy,
                   int64_t chunk, int64_t p, int64_t *owner)
{
    if (tm <= 0 || tn <= 0) return -1;
    int64_t ntiles = ((R + tm - 1) / tm) * ((Cn + tn - 1) / tn);
    return orc_owner_map(policy, chunk, ntiles, p, owner);
}

/* Executors of a tiled collapse(2) nest (reading c24; PAPER.md:622/666
 * tiling before parallelisation, Fig. 3 distribute teams / units):
 * tiles of BM x BN anchored at induction value 0 of each level cover the
 * space [lb0,ub0) x [lb1,ub1); tile id = row-major over the tiles that touch
 * the space; the tile loop runs over p_teams teams with (policy, chunk); the
 * BM*BN box positions of a tile (row-major) run over `units` units with
 * static chunk ic.  For box index t = tile*BM*BN + pos: team[t], unit[t] =
 * executor, or -1 where the box position is not an iteration.  Returns the
 * number of tiles, or -1. */
int64_t orc_tiled_owner_order(int64_t lb0, int64_t ub0, int64_t lb1, int64_t ub1, int64_t BM, int64_t BN,
                              int policy, int64_t chunk, int64_t p_teams, int64_t ic, int64_t units,
                              int order, int64_t *team, int64_t *unit);

int64_t orc_tiled_owner(int64_t lb0, int64_t ub0, int64_t lb1, int64_t ub1, int64_t BM, int64_t BN,
                        int policy, int64_t chunk, int64_t p_teams, int64_t ic, int64_t units,
                        int64_t *team, int64_t *unit)
{
    return orc_tiled_owner_order(lb0, ub0, lb1, ub1, BM, BN, policy, chunk, p_teams, ic, units, 0, team, unit);
}

/* As orc_tiled_owner, with the tile ids enumerated in another order (the
 * paper's tiling, fixes none).  order bit 0: column-major
 * (reading c35: tile id = (tj - tj0) * ntr + (ti - ti0)); order bit 1:
 * reversed (reading c38: id k is the tile the un-reversed order numbers
 * nt - 1 - k).  Arrays are indexed by that id. */
int64_t orc_tiled_owner_order(int64_t lb0, int64_t ub0, int64_t lb1, int64_t ub1, int64_t BM, int64_t BN,
                              int policy, int64_t chunk, int64_t p_teams, int64_t ic, int64_t units,
                              int order, int64_t *team, int64_t *unit)
{
    int colmajor = order & 1;
    if (BM <= 0 || BN <= 0 || ic <= 0 || units <= 0 || p_teams <= 0) return -1;
    if (ub0 <= lb0 || ub1 <= lb1) return 0;
    int64_t ti0 = lb0 / BM, tj0 = lb1 / BN;
    int64_t ntr = (ub0 + BM - 1) / BM - ti0, ntc = (ub1 + BN - 1) / BN - tj0;
    int64_t nt = ntr * ntc, P = BM * BN;
    int64_t *towner = (int64_t *)malloc(sizeof(int64_t) * (size_t)nt);
    if (!towner) return -1;
    if (orc_owner_map(policy, chunk, nt, p_teams, towner) != 0) { free(towner); return -1; }
    for (int64_t tile = 0; tile < nt; ++tile) {
        int64_t seq = (order & 2) ? nt - 1 - tile : tile;
        int64_t ti = colmajor ? ti0 + seq % ntr : ti0 + seq / ntc;
        int64_t tj = colmajor ? tj0 + seq / ntr : tj0 + seq % ntc;
        for (int64_t pos = 0; pos < P; ++pos) {
            int64_t i = ti * BM + pos / BN, j = tj * BN + pos % BN;
            int64_t t = tile * P + pos;
            if (i < lb0 || i >= ub0 || j < lb1 || j >= ub1) { team[t] = -1; unit[t] = -1; continue; }
            team[t] = towner[tile];
            unit[t] = (pos / ic) % units;          /* static, chunk ic over units */
        }
    }
    free(towner);
    return nt;
}

/* ---- matvec (PAPER.md:1217 'matrix-vector
 * multiplication', sizes PAPER.md:1405-1430) ----------------------------------
 * y[i] = sum_k A[i][k] * x[k] for i in [lb, ub), row-major A with leading
 * dimension lda, fp64 from the fp32 inputs; rows outside [lb, ub) keep y_in. */
int orc_matvec(int64_t M, int64_t K, int64_t lda, int64_t lb, int64_t ub, const float *A,
               const float *x, const double *y_in, double *y)
{
    if (lb < 0 || ub > M || lda < K) return -1;
    for (int64_t i = 0; i < M; ++i) y[i] = y_in[i];
    for (int64_t i = lb; i < ub; ++i) {
        double acc = 0.0;
        for (int64_t k = 0; k < K; ++k) acc += (double)A[i * lda + k] * (double)x[k];
        y[i] = acc;
    }
    return 0;
}

/* ---- 2-D filter stencil (the paper's "2D stencil,
 * filter size = 7", whose weights and boundary are unstated:
 * reading c28) -------------------------------------------------------------
 * out[i][j] = sum_{a,b in [-R,R]} w[a+R][b+R] * in[i+a][j+b] for
 * R <= i < ny-R, R <= j < nx-R; every other point copied unchanged.  S sweeps
 * ping-pong, fp64 from the fp32 initial grid and weights. */
int orc_stencil2d(int64_t ny, int64_t nx, int64_t R, int64_t S, const float *w, const float *init,
                  double *out)
{
    if (ny < 1 || nx < 1 || R < 0 || S < 0) return -1;
    int64_t F = 2 * R + 1;
    size_t N = (size_t)ny * (size_t)nx;
    double *a = (double *)malloc(N * sizeof(double));
    double *b = (double *)malloc(N * sizeof(double));
    if (!a || !b) { free(a); free(b); return -1; }
    for (size_t e = 0; e < N; ++e) a[e] = (double)init[e];
    memcpy(b, a, N * sizeof(double));
    for (int64_t s = 0; s < S; ++s) {
        for (int64_t i = R; i < ny - R; ++i)
            for (int64_t j = R; j < nx - R; ++j) {
                double acc = 0.0;
                for (int64_t p = 0; p < F; ++p)
                    for (int64_t q = 0; q < F; ++q)
                        acc += (double)w[p * F + q] * a[(i + p - R) * nx + (j + q - R)];
                b[i * nx + j] = acc;
            }
        double *t = a; a = b; b = t;
    }
    memcpy(out, a, N * sizeof(double));
    free(a); free(b);
    return 0;
}

/* ---- full-size reductions over the synthetic input stream -----------------
 * The oracle's own copy of the counter-based input recipe (DESIGN.md "Input
 * recipe"; the task allows each side its own implementation of the same
 * generator), fused with a plain sequential reduction so that 2^30 .. 2^34
 * element references need no host array.  dist 2 = i64 U[-2^28, 2^28),
 * dist 0 = f32 U[0,1).  Elements [start, start + n) of `stream`; result =
 * init (+) x_start (+) ... in index order (exact int64 / fp64). */
static uint64_t orc_mix(uint64_t z)
{
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

int orc_reduce_stream(int op, int dist, uint64_t stream, int64_t start, int64_t n, double *res_f,
                      int64_t *res_i)
{
    uint64_t seed = (2209ull << 16) | stream;
    if (dist == 2) {
        uint64_t acc = i64_identity(op);
        for (int64_t e = 0; e < n; ++e) {
            uint64_t x = orc_mix(seed + ((uint64_t)(start + e) + 1ull) * 0x9E3779B97F4A7C15ull);
            acc = i64_combine(op, acc, (int64_t)(x >> 35) - ((int64_t)1 << 28));
        }
        *res_i = (int64_t)acc;
        return 0;
    }
    if (dist == 0) {
        double acc = f_identity(op);
        for (int64_t e = 0; e < n; ++e) {
            uint64_t x = orc_mix(seed + ((uint64_t)(start + e) + 1ull) * 0x9E3779B97F4A7C15ull);
            acc = f_combine(op, acc, (double)(x >> 40) * 0x1.0p-24);
        }
        *res_f = acc;
        return 0;
    }
    return -1;
}
