import sys, os, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2209_10643_b200 as U
ctx = U.upir_init(0)
def run(A, B, dtype):
    M, K = A.shape; N = B.shape[1]
    if dtype == U.BF16:
        a = (A.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16); b = (B.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    else:
        a, b = A.astype(np.float32), B.astype(np.float32)
    C = np.full((M, N), -1.0, np.float32)
    ma = U.upir_data_map(ctx, a, U.MAP_TO); mb = U.upir_data_map(ctx, b, U.MAP_TO); mc = U.upir_data_map(ctx, C, U.MAP_TOFROM)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(1, 256 if dtype == U.BF16 else 384))
    U.upir_loop_exec(s, U.loop_desc([0, 0], [M, N], distribute=U.DIST_TEAMS), U.body(U.BODY_MATMUL, dtype, in0=ma, in1=mb, out=mc, ld=(K, N, N), dims=(K, M, N)))
    U.upir_spmd_end(s)
    for m in (mc, mb, ma): U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)
    return C
for dt in (U.BF16, U.F32):
    C = run(np.ones((128, 32)), np.ones((32, 256)), dt); print(dt, "ones", C[0, :4], C[127, 250:], np.unique(C)[:5])
    A = np.zeros((128, 32)); A[:, 0] = 1; B = np.arange(32 * 256).reshape(32, 256) % 7
    C = run(A, B, dt); print(dt, "row0 of B", C[0, :8], B[0, :8])
    A = np.zeros((128, 32)); A[:, 9] = 1
    C = run(A, B, dt); print(dt, "row9 of B", C[0, :8], B[9, :8])
    A = np.eye(128, 32); C = run(A, B, dt); print(dt, "eye", (C[:32] == B[:32]).mean(), C[5, :6], B[5, :6])
U.upir_finalize(ctx)
