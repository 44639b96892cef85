import sys, os, time, ctypes, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2209_10643_b200 as U
n = 1 << 30
ctx = U.upir_init(0)
hi = torch.empty(n, dtype=torch.int64, pin_memory=True)
hf = torch.empty(n, dtype=torch.float32, pin_memory=True)
hi.fill_(3); hf.fill_(1.0)
def arr(t, ct):
    return np.ctypeslib.as_array(ctypes.cast(t.data_ptr(), ctypes.POINTER(ct)), shape=(t.numel(),))
ai, af = arr(hi, ctypes.c_int64), arr(hf, ctypes.c_float)
res = np.zeros(8, np.float64)
# raw H2D bandwidth with torch
d = torch.empty(n, dtype=torch.int64, device="cuda")
torch.cuda.synchronize(); t = time.perf_counter(); d.copy_(hi, non_blocking=True); torch.cuda.synchronize()
print("torch H2D 8GiB pinned: %.1f GB/s" % (8 * 2**30 / (time.perf_counter() - t) / 1e9)); del d; torch.cuda.empty_cache()
for it in range(3):
    T = {}
    t0 = time.perf_counter()
    m1 = U.upir_data_map(ctx, ai, U.MAP_TO); U.upir_sync(ctx); T["map_i64"] = time.perf_counter() - t0
    t1 = time.perf_counter(); m2 = U.upir_data_map(ctx, af, U.MAP_TO); U.upir_sync(ctx); T["map_f32"] = time.perf_counter() - t1
    t1 = time.perf_counter(); mr = U.upir_data_map(ctx, res, U.MAP_FROM); rp, _, _ = U.upir_data_device_ptr(mr)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(592, 256))
    U.upir_loop_exec(s, U.loop_desc(0, n), U.body(U.BODY_REDUCE, U.I64, in0=m1), [U.reduction(U.OP_SUM, U.I64, rp), U.reduction(U.OP_MAX, U.I64, rp + 8)])
    U.upir_loop_exec(s, U.loop_desc(0, n), U.body(U.BODY_REDUCE, U.F32, in0=m2), [U.reduction(U.OP_SUM, U.F32, rp + 16), U.reduction(U.OP_MAX, U.F32, rp + 24)])
    U.upir_spmd_end(s); U.upir_sync(ctx); T["loops"] = time.perf_counter() - t1
    t1 = time.perf_counter(); U.upir_data_unmap(ctx, mr); U.upir_data_unmap(ctx, m2); U.upir_data_unmap(ctx, m1); U.upir_sync(ctx); T["unmap"] = time.perf_counter() - t1
    T["total"] = time.perf_counter() - t0
    print({k: round(v * 1e3, 1) for k, v in T.items()}, "GB/s", round(12 * 2**30 / T["total"] / 1e9, 1), res[:2])
U.upir_finalize(ctx)
