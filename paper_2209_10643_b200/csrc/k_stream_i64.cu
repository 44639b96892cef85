// Instantiation of the streaming loop kernels for body SB_RED_I64 (see k_stream.cuh).
#include "k_stream.cuh"

namespace upir {
cudaError_t launch_stream_i64(int nred, int path, int segv, int nst, bool trace, int teams, int units,
                            size_t smem, const StreamArgs &a, cudaStream_t s) {
  return launch_stream_body<SB_RED_I64>(nred, path, segv, nst, trace, teams, units, smem, a, s);
}
size_t staged_bytes_i64(int units, int segv, int nst) { return staged_bytes_body<SB_RED_I64>(units, segv, nst); }
}  // namespace upir
