"""B200-native runtime for the data-parallel hot path of UPIR (arXiv 2209.10643).

Python binding of the C-ABI in include/upir.h: the functions below carry the
C names and only marshal arguments (numpy arrays -> host pointers, torch CUDA
tensors -> device pointers, descriptors -> ctypes structs).  Every step of
the loop path runs in libupir.so's sm_100a kernels; nothing here computes.
"""
import ctypes

from . import _abi
from ._abi import *  # noqa: F401,F403  (enum values, structs, UpirError)
from ._abi import check, lib, UpirError  # noqa: F401

__all__ = [n for n in _abi.DECLARED] + ["loop_desc", "spmd_desc", "body", "reduction", "dist",
                                        "host_ptr", "dev_ptr"]


# ---- marshalling helpers --------------------------------------------------------
def host_ptr(a):
    """Host pointer and byte size of a C-contiguous numpy array."""
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("host array must be C-contiguous")
    return ctypes.c_void_p(a.ctypes.data), a.nbytes


def dev_ptr(t):
    """Device pointer of a torch CUDA tensor (or an int address)."""
    if isinstance(t, int):
        return ctypes.c_void_p(t)
    return ctypes.c_void_p(t.data_ptr())


def spmd_desc(num_teams, num_units, target=_abi.TARGET_GPU):
    return _abi.SpmdDesc(num_teams, num_units, target, 0)


def loop_desc(lb, ub, step=None, policy=_abi.SCHED_STATIC, chunk=0, distribute=_abi.DIST_TEAMS_UNITS,
              tile=None, inner_policy=_abi.SCHED_STATIC, inner_chunk=0, flags=0, simdlen=0):
    lb = list(lb) if isinstance(lb, (list, tuple)) else [lb]
    ub = list(ub) if isinstance(ub, (list, tuple)) else [ub]
    n = len(lb)
    step = [1] * n if step is None else (list(step) if isinstance(step, (list, tuple)) else [step])
    tile = [0] * n if tile is None else list(tile)
    pad = lambda v: (ctypes.c_int64 * 3)(*(v + [0] * (3 - len(v))))  # noqa: E731
    d = _abi.LoopDesc()
    d.collapse = n
    d.policy = policy
    d.lb, d.ub, d.step, d.tile = pad(lb), pad(ub), pad(step), pad(tile)
    d.chunk = chunk
    d.distribute = distribute
    d.inner_policy = inner_policy
    d.inner_chunk = inner_chunk
    d.flags = flags
    d.simdlen = simdlen
    return d


def body(kind, dtype, in0=None, in1=None, out=None, alpha=0.0, ld=(0, 0, 0), dims=(0, 0, 0)):
    b = _abi.Body()
    b.kind, b.dtype = kind, dtype
    b.in0, b.in1, b.out = in0, in1, out
    b.alpha = alpha
    b.ld = (ctypes.c_int64 * 3)(*ld)
    b.dims = (ctypes.c_int64 * 3)(*dims)
    return b


def reduction(op, dtype, dev_result, init=None):
    """init: None (identity) or a Python number; kept alive on the struct."""
    r = _abi.Reduction()
    r.op, r.dtype = op, dtype
    r.dev_result = dev_ptr(dev_result).value
    if init is not None:
        if hasattr(init, "item"):   # numpy scalar / one-element array
            init = init.item() if getattr(init, "size", 1) == 1 else init
        buf = (ctypes.c_int64(int(init)) if dtype == _abi.I64 else ctypes.c_float(float(init)))
        r._init_buf = buf
        r.init = ctypes.cast(ctypes.pointer(buf), ctypes.c_void_p)
    return r


def dist(n_rows, row_elems, elem_bytes, halo_rows=0, pattern=_abi.PATTERN_BLOCK):
    return _abi.Dist(pattern, halo_rows, n_rows, row_elems, elem_bytes)


# ---- C entry points (same names) --------------------------------------------------
def upir_version():
    return lib().upir_version().decode()


def upir_last_error():
    return lib().upir_last_error().decode()


def upir_init(device=0, rank=0, nranks=1, nccl_id=None, compute_stream=0, copy_stream=0):
    ctx = ctypes.c_void_p()
    if nranks == 1 and not compute_stream and not copy_stream:
        check(lib().upir_init(device, None, ctypes.byref(ctx)))
    else:
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
        w = _abi.World(rank, nranks, ctypes.cast(idbuf, ctypes.c_void_p) if idbuf else None,
                       compute_stream, copy_stream)
        check(lib().upir_init(device, ctypes.byref(w), ctypes.byref(ctx)))
    return ctx


def upir_finalize(ctx):
    check(lib().upir_finalize(ctx))


def upir_comm_unique_id():
    buf = ctypes.create_string_buffer(128)
    check(lib().upir_comm_unique_id(buf))
    return bytes(buf.raw)


def upir_ctx_stream(ctx, which=0):
    s = ctypes.c_size_t()
    check(lib().upir_ctx_stream(ctx, which, ctypes.byref(s)))
    return s.value


def upir_ctx_stats(ctx):
    out = (ctypes.c_int64 * 4)()
    check(lib().upir_ctx_stats(ctx, out))
    return {"h2d_bytes": out[0], "d2h_bytes": out[1], "live_maps": out[2], "launches": out[3]}


def upir_data_map(ctx, host_array, kind, dist_=None):
    p, n = host_ptr(host_array)
    m = ctypes.c_void_p()
    check(lib().upir_data_map(ctx, p, n, kind, ctypes.byref(dist_) if dist_ is not None else None,
                              ctypes.byref(m)))
    return m


def upir_data_adopt(ctx, tensor, dist_=None, nbytes=None):
    m = ctypes.c_void_p()
    nb = nbytes if nbytes is not None else tensor.numel() * tensor.element_size()
    check(lib().upir_data_adopt(ctx, dev_ptr(tensor), nb, ctypes.byref(dist_) if dist_ is not None else None,
                                ctypes.byref(m)))
    return m


def upir_data_unmap(ctx, m):
    check(lib().upir_data_unmap(ctx, m))


def upir_data_update(ctx, m, direction):
    check(lib().upir_data_update(ctx, m, direction))


def upir_data_update_section(ctx, m, byte_offset, nbytes, direction):
    check(lib().upir_data_update_section(ctx, m, byte_offset, nbytes, direction))


def upir_data_device_ptr(m):
    p, n, off = ctypes.c_void_p(), ctypes.c_int64(), ctypes.c_int64()
    check(lib().upir_data_device_ptr(m, ctypes.byref(p), ctypes.byref(n), ctypes.byref(off)))
    return p.value, n.value, off.value


def upir_dist_owned_rows(n_rows, rank, nranks):
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    check(lib().upir_dist_owned_rows(n_rows, rank, nranks, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def upir_halo_plan(n_rows, halo_rows, rank, nranks):
    out = (ctypes.c_int64 * 8)()
    check(lib().upir_halo_plan(n_rows, halo_rows, rank, nranks, out))
    return {"send_up": (out[0], out[1]), "recv_up": (out[2], out[3]),
            "send_dn": (out[4], out[5]), "recv_dn": (out[6], out[7])}


def upir_spmd_launch(ctx, desc):
    s = ctypes.c_void_p()
    check(lib().upir_spmd_launch(ctx, ctypes.byref(desc), ctypes.byref(s)))
    return s


def upir_spmd_end(s):
    check(lib().upir_spmd_end(s))


def _reds(reds):
    reds = list(reds or [])
    if not reds:
        return None, 0, None
    arr = (_abi.Reduction * len(reds))(*reds)
    return arr, len(reds), reds


def upir_loop_exec(spmd, loop, body_, reds=None, trace=None):
    arr, n, keep = _reds(reds)
    check(lib().upir_loop_exec(spmd, ctypes.byref(loop), ctypes.byref(body_), arr, n, trace))


def upir_loop_normalize(loop):
    T = ctypes.c_int64()
    Td = (ctypes.c_int64 * 3)()
    check(lib().upir_loop_normalize(ctypes.byref(loop), ctypes.byref(T), Td))
    return T.value, tuple(Td)


def upir_loop_validate(spmd, loop, body_kind, reds=None):
    arr, n, keep = _reds(reds)
    return lib().upir_loop_validate(ctypes.byref(spmd), ctypes.byref(loop), body_kind, arr, n)


def upir_schedule_chunks(policy, chunk, T, p, u):
    cap = 1
    while True:
        lo = (ctypes.c_int64 * cap)()
        hi = (ctypes.c_int64 * cap)()
        cnt = ctypes.c_int64()
        check(lib().upir_schedule_chunks(policy, chunk, T, p, u, lo, hi, cap, ctypes.byref(cnt)))
        if cnt.value <= cap:
            return [(lo[i], hi[i]) for i in range(cnt.value)]
        cap = cnt.value


def upir_reduce(ctx, op, dtype, dev_in, count, dev_out, scope=_abi.SCOPE_DEVICE):
    check(lib().upir_reduce(ctx, op, dtype, dev_ptr(dev_in), count, dev_ptr(dev_out), scope))


def upir_reduce_async(ctx, op, dtype, dev_in, count, dev_out):
    """WORLD allreduce as async arrive-compute; returns the token for
    upir_sync(JOIN / WAIT)."""
    tok = ctypes.c_void_p()
    check(lib().upir_reduce_async(ctx, op, dtype, dev_ptr(dev_in), count, dev_ptr(dev_out), ctypes.byref(tok)))
    return tok


def upir_sync(ctx, kind=_abi.SYNC_BARRIER, halo_map=None, token=None, async_=False):
    """Returns the token (ARRIVE, async HALO).  HALO is synchronous unless
    async_=True (then the C call receives a token out-param)."""
    if kind == _abi.SYNC_HALO and not async_:
        check(lib().upir_sync(ctx, kind, halo_map, None))
        return None
    tok = token if token is not None else ctypes.c_void_p()
    check(lib().upir_sync(ctx, kind, halo_map, ctypes.byref(tok)))
    return tok


def upir_graph_begin(ctx):
    check(lib().upir_graph_begin(ctx))


def upir_graph_end(ctx):
    g = ctypes.c_void_p()
    check(lib().upir_graph_end(ctx, ctypes.byref(g)))
    return g


def upir_graph_launch(ctx, g):
    check(lib().upir_graph_launch(ctx, g))


def upir_graph_destroy(g):
    check(lib().upir_graph_destroy(g))


def upir_synth_fill(ctx, m, dist_kind, stream, index_base=0, n_rows=0, n_cols=0):
    check(lib().upir_synth_fill(ctx, m, dist_kind, stream, index_base, n_rows, n_cols))


def upir_peer_export(ctx, m=None):
    """Peer record (bytes) of the context window (m None) or of map m."""
    buf = ctypes.create_string_buffer(_abi.PEER_REC_BYTES)
    check(lib().upir_peer_export(ctx, m, buf))
    return bytes(buf.raw)


def upir_peer_import(ctx, m, peer_rank, rec):
    buf = ctypes.create_string_buffer(bytes(rec), _abi.PEER_REC_BYTES)
    check(lib().upir_peer_import(ctx, m, peer_rank, buf))


def upir_peer_share(ctx, maps=(), group=None):
    """Collective over torch.distributed: export this rank's window and maps,
    all-gather the records, import every rank's window and the halo
    neighbours' (rank +- 1) map buffers.  Host plumbing only."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    recs = [upir_peer_export(ctx, None)] + [upir_peer_export(ctx, m) for m in maps]
    allr = [None] * world
    dist.all_gather_object(allr, (rank, recs), group=group)
    for q, rr in allr:
        upir_peer_import(ctx, None, q, rr[0])
        if abs(q - rank) == 1:
            for k, m in enumerate(maps):
                upir_peer_import(ctx, m, q, rr[k + 1])
