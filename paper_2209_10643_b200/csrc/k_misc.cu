// k_misc.cu -- dispatch of the streaming bodies, the ordered rank combine of
// upir_reduce(WORLD), and the device-side synthetic input generator.
#include <math_constants.h>

#include "dev_peer.cuh"
#include "upir_internal.h"

namespace upir {

cudaError_t launch_stream_i64(int, int, int, int, bool, int, int, size_t, const StreamArgs &, cudaStream_t);
cudaError_t launch_stream_f32(int, int, int, int, bool, int, int, size_t, const StreamArgs &, cudaStream_t);
cudaError_t launch_stream_axpy(int, int, int, int, bool, int, int, size_t, const StreamArgs &, cudaStream_t);
size_t staged_bytes_i64(int, int, int);
size_t staged_bytes_f32(int, int, int);
size_t staged_bytes_axpy(int, int, int);

cudaError_t launch_stream_loop(int body, int path, int segv, int nst, bool trace, int teams, int units,
                               size_t smem, const StreamArgs &a, cudaStream_t s) {
  switch (body) {
    case SB_RED_I64: return launch_stream_i64(a.nred, path, segv, nst, trace, teams, units, smem, a, s);
    case SB_RED_F32: return launch_stream_f32(a.nred, path, segv, nst, trace, teams, units, smem, a, s);
    case SB_AXPY: return launch_stream_axpy(a.nred, path, segv, nst, trace, teams, units, smem, a, s);
  }
  return cudaErrorInvalidValue;
}

size_t staged_smem_bytes(int body, int units, int segv, int nst) {
  switch (body) {
    case SB_RED_I64: return staged_bytes_i64(units, segv, nst);
    case SB_RED_F32: return staged_bytes_f32(units, segv, nst);
    case SB_AXPY: return staged_bytes_axpy(units, segv, nst);
  }
  return 0;
}

// ---- upir_reduce(WORLD): ordered combine of gathered per-rank values --------
// gathered: [nranks][count]; out[e] = g[0][e] (+) g[1][e] (+) ... in ascending
// rank order (reading c10; oracle o8).  fp32 values are combined in fp64 and
// rounded once.
__global__ void rank_combine_kernel(int op, int dtype, const void *gathered, int64_t count, int nranks,
                                    void *out) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < count;
       e += (int64_t)gridDim.x * blockDim.x) {
    if (dtype == UPIR_I64) {
      const long long *g = reinterpret_cast<const long long *>(gathered);
      unsigned long long acc = (unsigned long long)g[e];
      for (int r = 1; r < nranks; ++r) {
        const long long v = g[(int64_t)r * count + e];
        if (op == UPIR_OP_SUM) acc += (unsigned long long)v;
        else if (op == UPIR_OP_MAX) acc = ((long long)acc > v) ? acc : (unsigned long long)v;
        else acc = ((long long)acc < v) ? acc : (unsigned long long)v;
      }
      reinterpret_cast<long long *>(out)[e] = (long long)acc;
    } else {
      const float *g = reinterpret_cast<const float *>(gathered);
      double acc = g[e];
      for (int r = 1; r < nranks; ++r) {
        const double v = g[(int64_t)r * count + e];
        if (op == UPIR_OP_SUM) acc += v;
        else if (op == UPIR_OP_MAX) acc = fmax(acc, v);
        else acc = fmin(acc, v);
      }
      reinterpret_cast<float *>(out)[e] = (float)acc;
    }
  }
}

struct WorldCombineArgs { RedSpec red[2]; };
__global__ void world_combine_kernel(const unsigned long long *g, int nranks, int nred, WorldCombineArgs w) {
  for (int r = 0; r < nred; ++r) {
    const RedSpec &rs = w.red[r];
    if (rs.dtype == UPIR_I64) {
      unsigned long long acc = rs.init_bits;
      for (int q = 0; q < nranks; ++q) {
        const long long v = (long long)g[q * 2 + r];
        if (rs.op == UPIR_OP_SUM) acc += (unsigned long long)v;
        else if (rs.op == UPIR_OP_MAX) acc = ((long long)acc > v) ? acc : (unsigned long long)v;
        else acc = ((long long)acc < v) ? acc : (unsigned long long)v;
      }
      *reinterpret_cast<long long *>(rs.result) = (long long)acc;
    } else {
      double acc = __longlong_as_double((long long)rs.init_bits);
      for (int q = 0; q < nranks; ++q) {
        const double v = __longlong_as_double((long long)g[q * 2 + r]);
        if (rs.op == UPIR_OP_SUM) acc += v;
        else if (rs.op == UPIR_OP_MAX) acc = fmax(acc, v);
        else acc = fmin(acc, v);
      }
      *reinterpret_cast<float *>(rs.result) = (float)acc;   // the one rounding
    }
  }
}

cudaError_t launch_world_combine(const unsigned long long *gathered, int nranks, int nred, const RedSpec *reds,
                                 cudaStream_t s) {
  WorldCombineArgs w;
  for (int r = 0; r < 2; ++r) w.red[r] = r < nred ? reds[r] : RedSpec{};
  world_combine_kernel<<<1, 1, 0, s>>>(gathered, nranks, nred, w);
  return cudaGetLastError();
}

cudaError_t launch_rank_combine(int op, int dtype, const void *gathered, int64_t count, int nranks,
                                void *out, cudaStream_t s) {
  const int threads = 256;
  int64_t blocks = (count + threads - 1) / threads;
  if (blocks > 1184) blocks = 1184;
  if (blocks < 1) blocks = 1;
  rank_combine_kernel<<<(int)blocks, threads, 0, s>>>(op, dtype, gathered, count, nranks, out);
  return cudaGetLastError();
}

// ---- peer mode: drain the neighbours' deliveries ---------------------------
__global__ void peer_drain_kernel(unsigned long long *win, int has_up, int has_dn) {
  const unsigned long long g = *reinterpret_cast<volatile unsigned long long *>(win + WIN_HALO_GEN);
  if (has_up) wait_geq_sys(win + WIN_HALO_FROM_UP, g);
  if (has_dn) wait_geq_sys(win + WIN_HALO_FROM_DN, g);
}

cudaError_t launch_peer_drain(unsigned long long *win, int has_up, int has_dn, cudaStream_t s) {
  peer_drain_kernel<<<1, 1, 0, s>>>(win, has_up, has_dn);
  return cudaGetLastError();
}

__global__ void peer_barrier_kernel(unsigned long long *win, int nranks) {
  const unsigned long long e = *reinterpret_cast<volatile unsigned long long *>(win + WIN_BAR_GEN);
  for (int q = 0; q < nranks; ++q)
    red_release_sys_add(reinterpret_cast<unsigned long long *>(win[WIN_PEERS + q]) + WIN_BAR_CNT, 1ull);
  wait_geq_sys(win + WIN_BAR_CNT, (e + 1ull) * (unsigned long long)nranks);
  *reinterpret_cast<volatile unsigned long long *>(win + WIN_BAR_GEN) = e + 1ull;
}

cudaError_t launch_peer_barrier(unsigned long long *win, int nranks, cudaStream_t s) {
  peer_barrier_kernel<<<1, 1, 0, s>>>(win, nranks);
  return cudaGetLastError();
}

// the CTA copies n bytes (16-B vectors when both ends and n allow)
__device__ __forceinline__ void copy_bytes_all(char *dst, const char *src, int64_t n) {
  if ((((uintptr_t)dst | (uintptr_t)src | (uintptr_t)n) & 15) == 0) {
    uint4 *d = reinterpret_cast<uint4 *>(dst);
    const uint4 *s = reinterpret_cast<const uint4 *>(src);
    for (int64_t e = threadIdx.x; e < n / 16; e += blockDim.x) d[e] = s[e];
  } else {
    for (int64_t e = threadIdx.x; e < n; e += blockDim.x) dst[e] = src[e];
  }
}

// ---- upir_reduce(WORLD) over the peer windows -------------------------------
// Generation e = peer allreduces this rank completed; its staging half is
// e & 1.  Every rank: stage dev_in, publish (release add on every window's
// arrival counter), wait for (e + 1) * N arrivals (acquire), combine rank 0,
// 1, ... N-1 element-wise exactly as rank_combine_kernel (fp32 in fp64,
// rounded once).  Staging half e & 1 is rewritten at generation e + 2 only:
// by then every rank has arrived at e + 1, i.e. finished reading it at e.
__global__ void __launch_bounds__(1024) peer_allreduce_kernel(unsigned long long *win, int nranks, int op, int dtype,
                                                              const void *dev_in, int64_t count, void *dev_out) {
  __shared__ unsigned long long e;
  if (threadIdx.x == 0) e = *reinterpret_cast<volatile unsigned long long *>(win + WIN_AR_GEN);
  __syncthreads();
  const int64_t half = (int64_t)(e & 1ull) * WIN_AR_ELEMS * 8;
  const int esz = dtype == UPIR_I64 ? 8 : 4;
  copy_bytes_all(reinterpret_cast<char *>(win) + WIN_AR_OFF + half, reinterpret_cast<const char *>(dev_in),
                 count * esz);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int q = 0; q < nranks; ++q)
      red_release_sys_add(reinterpret_cast<unsigned long long *>(win[WIN_PEERS + q]) + WIN_AR_CNT, 1ull);
    wait_geq_sys(win + WIN_AR_CNT, (e + 1ull) * (unsigned long long)nranks);
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < count; i += blockDim.x) {
    auto staged = [&](int q) {
      return reinterpret_cast<const char *>(win[WIN_PEERS + q]) + WIN_AR_OFF + half;
    };
    if (dtype == UPIR_I64) {
      unsigned long long acc = (unsigned long long)reinterpret_cast<const long long *>(staged(0))[i];
      for (int q = 1; q < nranks; ++q) {
        const long long v = reinterpret_cast<const long long *>(staged(q))[i];
        if (op == UPIR_OP_SUM) acc += (unsigned long long)v;
        else if (op == UPIR_OP_MAX) acc = ((long long)acc > v) ? acc : (unsigned long long)v;
        else acc = ((long long)acc < v) ? acc : (unsigned long long)v;
      }
      reinterpret_cast<long long *>(dev_out)[i] = (long long)acc;
    } else {
      double acc = reinterpret_cast<const float *>(staged(0))[i];
      for (int q = 1; q < nranks; ++q) {
        const double v = reinterpret_cast<const float *>(staged(q))[i];
        if (op == UPIR_OP_SUM) acc += v;
        else if (op == UPIR_OP_MAX) acc = fmax(acc, v);
        else acc = fmin(acc, v);
      }
      reinterpret_cast<float *>(dev_out)[i] = (float)acc;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) *reinterpret_cast<volatile unsigned long long *>(win + WIN_AR_GEN) = e + 1ull;
}

cudaError_t launch_peer_allreduce(unsigned long long *win, int nranks, int op, int dtype, const void *dev_in,
                                  int64_t count, void *dev_out, cudaStream_t s) {
  peer_allreduce_kernel<<<1, 1024, 0, s>>>(win, nranks, op, dtype, dev_in, count, dev_out);
  return cudaGetLastError();
}

// ---- upir_sync(HALO) over peer mappings ------------------------------------
// Generation g = exchanges + fused peer-mode sweeps this rank completed (the
// fused sweeps' counter, so both kinds interleave).  (1) Wait until both
// neighbours completed generation g - 1: they are done reading the halo rows
// I overwrite (their previous use of this buffer ended before their
// exchange g - 1 began).  (2) Store my boundary rows into their halo rows.
// (3) Publish: system-scope fence, release-add on their delivery counters.
// (4) Wait until both delivered generation g into my halo rows (acquire),
// then count the generation.
__global__ void __launch_bounds__(1024) peer_halo_kernel(PeerHaloArgs a) {
  __shared__ unsigned long long g;
  if (threadIdx.x == 0) {
    g = *reinterpret_cast<volatile unsigned long long *>(a.win + WIN_HALO_GEN);
    if (a.win_up) wait_geq_sys(a.win + WIN_HALO_FROM_UP, g);
    if (a.win_dn) wait_geq_sys(a.win + WIN_HALO_FROM_DN, g);
  }
  __syncthreads();
  if (a.win_up) copy_bytes_all(a.dst_up, a.src_up, a.bytes_up);
  if (a.win_dn) copy_bytes_all(a.dst_dn, a.src_dn, a.bytes_dn);
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (a.win_up) red_release_sys_add(a.win_up + WIN_HALO_FROM_DN, 1ull);
    if (a.win_dn) red_release_sys_add(a.win_dn + WIN_HALO_FROM_UP, 1ull);
    if (a.win_up) wait_geq_sys(a.win + WIN_HALO_FROM_UP, g + 1ull);
    if (a.win_dn) wait_geq_sys(a.win + WIN_HALO_FROM_DN, g + 1ull);
    fence_proxy_async_global();   // later TMA reads of the halo rows see the delivery
    *reinterpret_cast<volatile unsigned long long *>(a.win + WIN_HALO_GEN) = g + 1ull;
  }
}

cudaError_t launch_peer_halo(const PeerHaloArgs &a, cudaStream_t s) {
  peer_halo_kernel<<<1, 1024, 0, s>>>(a);
  return cudaGetLastError();
}

// ---- synthetic inputs: counter-based splitmix64 -
// An implementation of the recipe independent of synth/ (host numpy).
__device__ __forceinline__ unsigned long long sm_mix(unsigned long long z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void synth_fill_kernel(int dist, unsigned long long seed, void *dst, int64_t n, int64_t index0,
                                  int64_t n_rows, int64_t n_cols) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const unsigned long long gi = (unsigned long long)(index0 + e);
    const unsigned long long x = sm_mix(seed + (gi + 1ull) * 0x9E3779B97F4A7C15ull);
    switch (dist) {
      case 0:  // f32 U[0,1) on the 2^-24 grid
        reinterpret_cast<float *>(dst)[e] = (float)(x >> 40) * 0x1.0p-24f;
        break;
      case 1:  // f32 U[-1,1)
        reinterpret_cast<float *>(dst)[e] = 2.0f * ((float)(x >> 40) * 0x1.0p-24f) - 1.0f;
        break;
      case 2:  // i64 U[-2^28, 2^28)
        reinterpret_cast<long long *>(dst)[e] = (long long)(x >> 35) - (1ll << 28);
        break;
      case 3: {  // bf16 U[-1,1) on the 2^-6 grid (exact)
        const float f = ((float)(x >> 57) * 0x1.0p-7f) * 2.0f - 1.0f;
        const unsigned int bits = __float_as_uint(f);
        reinterpret_cast<unsigned short *>(dst)[e] = (unsigned short)(bits >> 16);
        break;
      }
      case 4: {  // Jacobi initial grid: interior U[0,1), top row 1, other boundary 0
        const int64_t i = (int64_t)gi / n_cols, j = (int64_t)gi % n_cols;
        float v = (float)(x >> 40) * 0x1.0p-24f;
        if (i == 0) v = 1.0f;
        else if (i == n_rows - 1 || j == 0 || j == n_cols - 1) v = 0.0f;
        reinterpret_cast<float *>(dst)[e] = v;
        break;
      }
    }
  }
}

cudaError_t launch_synth_fill(int dist, uint64_t stream, void *dst, int64_t n, int64_t index0, int64_t n_rows,
                              int64_t n_cols, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  const unsigned long long seed = (2209ull << 16) | (unsigned long long)stream;
  const int threads = 256;
  int64_t blocks = (n + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;
  synth_fill_kernel<<<(int)blocks, threads, 0, s>>>(dist, seed, dst, n, index0, n_rows, n_cols);
  return cudaGetLastError();
}

}  // namespace upir
