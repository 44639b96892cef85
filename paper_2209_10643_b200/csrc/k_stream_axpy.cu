// Instantiation of the streaming loop kernels for body SB_AXPY (see k_stream.cuh).
#include "k_stream.cuh"

namespace upir {
cudaError_t launch_stream_axpy(int nred, int path, int segv, int nst, bool trace, int teams, int units,
                            size_t smem, const StreamArgs &a, cudaStream_t s) {
  return launch_stream_body<SB_AXPY>(nred, path, segv, nst, trace, teams, units, smem, a, s);
}
size_t staged_bytes_axpy(int units, int segv, int nst) { return staged_bytes_body<SB_AXPY>(units, segv, nst); }
}  // namespace upir
