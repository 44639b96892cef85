"""ctypes mirror of include/upir.h (argument marshalling only).

Every call goes straight to libupir.so; there is no Python or CPU fallback:
if the library is missing or cannot initialise a device, the call raises.
"""
import ctypes
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libupir.so")

# ---- enums (values of include/upir.h) ----------------------------------------
OK, E_INVALID, E_UNSUPPORTED, E_NOT_MAPPED, E_OOM, E_CUDA, E_NCCL, E_SYNC, E_LEAK = range(9)
STATUS_NAMES = {0: "OK", 1: "E_INVALID", 2: "E_UNSUPPORTED", 3: "E_NOT_MAPPED", 4: "E_OOM",
                5: "E_CUDA", 6: "E_NCCL", 7: "E_SYNC", 8: "E_LEAK"}
I32, I64, F32, F64, BF16 = 0, 1, 2, 3, 4
MAP_TO, MAP_FROM, MAP_TOFROM, MAP_ALLOC = 1, 2, 3, 4
PATTERN_NONE, PATTERN_BLOCK = 0, 1
TARGET_GPU, TARGET_CLUSTER = 1, 2
SCHED_STATIC, SCHED_DYNAMIC, SCHED_GUIDED, SCHED_RUNTIME, SCHED_AUTO = 0, 1, 2, 3, 4
DIST_TEAMS, DIST_UNITS, DIST_TEAMS_UNITS = 1, 2, 3
NOWAIT = 1
WORLD_REDUCE = 2
TILE_COLMAJOR = 4
WORLD_VIA_COMM = 8
TILE_REVERSE = 16
HALO_EXPLICIT = 32
PEER_REC_BYTES = 256
BODY_AXPY, BODY_REDUCE, BODY_JACOBI5, BODY_MATMUL, BODY_MATVEC, BODY_STENCIL2D = 0, 1, 2, 3, 4, 5
OP_SUM, OP_MAX, OP_MIN = 0, 1, 2
SCOPE_DEVICE, SCOPE_WORLD = 0, 1
SYNC_BARRIER, SYNC_WORLD_BARRIER, SYNC_ARRIVE, SYNC_WAIT, SYNC_HALO, SYNC_JOIN = 0, 1, 2, 3, 4, 5
UPDATE_FORWARD, UPDATE_BACKWARD, UPDATE_FORWARD_ASYNC = 0, 1, 2

i32, i64, u32, u64 = ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
vp = ctypes.c_void_p


class World(ctypes.Structure):
    _fields_ = [("rank", i32), ("nranks", i32), ("nccl_id", vp),
                ("compute_stream", ctypes.c_size_t), ("copy_stream", ctypes.c_size_t)]


class Dist(ctypes.Structure):
    _fields_ = [("pattern", i32), ("halo_rows", i32), ("n_rows", i64), ("row_elems", i64),
                ("elem_bytes", i64)]


class SpmdDesc(ctypes.Structure):
    _fields_ = [("num_teams", i32), ("num_units", i32), ("target", u32), ("reserved", u32)]


class LoopDesc(ctypes.Structure):
    _fields_ = [("collapse", i32), ("policy", i32), ("lb", i64 * 3), ("ub", i64 * 3),
                ("step", i64 * 3), ("tile", i64 * 3), ("chunk", i64), ("distribute", i32),
                ("inner_policy", i32), ("inner_chunk", i64), ("flags", u32), ("simdlen", u32)]


class Body(ctypes.Structure):
    _fields_ = [("kind", i32), ("dtype", i32), ("in0", vp), ("in1", vp), ("out", vp),
                ("alpha", ctypes.c_double), ("ld", i64 * 3), ("dims", i64 * 3)]


class Reduction(ctypes.Structure):
    _fields_ = [("op", i32), ("dtype", i32), ("init", vp), ("dev_result", vp)]


_SIGS = {
    "upir_last_error": (ctypes.c_char_p, []),
    "upir_version": (ctypes.c_char_p, []),
    "upir_init": (i32, [ctypes.c_int, ctypes.POINTER(World), ctypes.POINTER(vp)]),
    "upir_finalize": (i32, [vp]),
    "upir_comm_unique_id": (i32, [vp]),
    "upir_ctx_stream": (i32, [vp, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]),
    "upir_ctx_stats": (i32, [vp, ctypes.POINTER(i64)]),
    "upir_data_map": (i32, [vp, vp, ctypes.c_size_t, ctypes.c_int, ctypes.POINTER(Dist), ctypes.POINTER(vp)]),
    "upir_data_adopt": (i32, [vp, vp, ctypes.c_size_t, ctypes.POINTER(Dist), ctypes.POINTER(vp)]),
    "upir_data_unmap": (i32, [vp, vp]),
    "upir_data_update": (i32, [vp, vp, ctypes.c_int]),
    "upir_data_update_section": (i32, [vp, vp, i64, i64, ctypes.c_int]),
    "upir_data_device_ptr": (i32, [vp, ctypes.POINTER(vp), ctypes.POINTER(i64), ctypes.POINTER(i64)]),
    "upir_dist_owned_rows": (i32, [i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]),
    "upir_halo_plan": (i32, [i64, i32, i32, i32, ctypes.POINTER(i64)]),
    "upir_spmd_launch": (i32, [vp, ctypes.POINTER(SpmdDesc), ctypes.POINTER(vp)]),
    "upir_spmd_end": (i32, [vp]),
    "upir_loop_exec": (i32, [vp, ctypes.POINTER(LoopDesc), ctypes.POINTER(Body), ctypes.POINTER(Reduction),
                             i32, vp]),
    "upir_loop_normalize": (i32, [ctypes.POINTER(LoopDesc), ctypes.POINTER(i64), ctypes.POINTER(i64)]),
    "upir_loop_validate": (i32, [ctypes.POINTER(SpmdDesc), ctypes.POINTER(LoopDesc), i32,
                                 ctypes.POINTER(Reduction), i32]),
    "upir_schedule_chunks": (i32, [i32, i64, i64, i64, i64, ctypes.POINTER(i64), ctypes.POINTER(i64), i64,
                                   ctypes.POINTER(i64)]),
    "upir_reduce": (i32, [vp, i32, i32, vp, i64, vp, i32]),
    "upir_reduce_async": (i32, [vp, i32, i32, vp, i64, vp, vp]),
    "upir_sync": (i32, [vp, i32, vp, ctypes.POINTER(vp)]),
    "upir_graph_begin": (i32, [vp]),
    "upir_graph_end": (i32, [vp, ctypes.POINTER(vp)]),
    "upir_graph_launch": (i32, [vp, vp]),
    "upir_graph_destroy": (i32, [vp]),
    "upir_synth_fill": (i32, [vp, vp, i32, u64, i64, i64, i64]),
    "upir_peer_export": (i32, [vp, vp, vp]),
    "upir_peer_import": (i32, [vp, vp, i32, vp]),
}

DECLARED = tuple(_SIGS)

_lib = None


class UpirError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def lib():
    """Load libupir.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(python -m paper_2209_10643_b200.build); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status):
    if status != OK:
        raise UpirError(status, lib().upir_last_error().decode())
    return status
