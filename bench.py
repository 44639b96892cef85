"""Benchmark of the UPIR data-parallel loop path on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl upir|reference]
                    [--workload reduce|axpy|jacobi|matmul] [--sched static|static1|dynamic]

For N > 1 launch under torchrun (one rank per GPU, NCCL).  Rank 0 prints ONE
JSON line.  Default workload = BASELINE.json configs[1]: int64 and fp32
sum/max reduction over n = 2^30 elements per GPU, teams x units = 148*4 x 256
SPMD region, worksharing loop under schedule(static) with the two reductions
fused into the loop (one pass per array), map to/from; at N > 1 each rank
reduces its own 2^30-element arrays and the four results are combined over
ranks with upir_reduce(WORLD) (weak scaling).

A step = one pass of the whole path over the step's input:
  value : the loop kernels + world combine with inputs resident in HBM
  e2e   : through the C-ABI with HOST buffers -- upir_data_map(TO) of the
          pinned host arrays (H2D), the loops, the world combine, the result
          scalars mapped FROM (D2H) and unmap, every step.
Inputs (12 GiB per GPU) are far larger than L2 (126 MB): no flush needed.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

GIB = 1 << 30


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="upir", choices=["upir", "reference"])
    ap.add_argument("--workload", default="reduce", choices=["reduce", "reduce34", "jacobi32k"],
                    help="reduce = C2 (default); reduce34 = C5a 2^34 int64 strong scaling; "
                         "jacobi32k = C5b 32768^2 Jacobi with halo exchange, strong scaling")
    ap.add_argument("--sched", default=None, choices=["static", "static1", "dynamic"],
                    help="default: static for C2; static1 (one 16-B vector per chunk) for C5a, whose 2^34-element "
                         "static blocks put ~65k distinct 2 MB pages in flight (TLB-bound, see DESIGN.md)")
    ap.add_argument("--n-log2", type=int, default=30)
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-kernels", action="store_true", help="skip the axpy / Jacobi / matmul kernel lines")
    return ap.parse_args()


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [v.strip() for v in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def ncu_traffic(kernel_key):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d.get(kernel_key)
    return None


# --------------------------------------------------------------------------- dist
def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


C2_METRIC = "GB/s per upir.loop reduction (int64+fp32 sum/max, n=2^30 per GPU)"


def c2_config(sched, world):
    return {"workload": "C2: int64 and fp32 sum/max reduction, n=2^30 per GPU, teams x units 592x256, "
                        f"schedule {sched}, map to/from",
            "teams": 592, "units": 256, "schedule": sched,
            "l2": "inputs 12 GiB per GPU >> 126 MB L2 (no flush needed)", "parallelism": f"dp{world}"}


# --------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle (plain sequential CPU interpreter) as the reference arm, on a
    bounded sample of the same workload, timed on this host's cores."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    import synth
    n = 1 << 24
    xi = synth.c_i64_sym(6, 0, n)
    xf = synth.c_f32_unit(7, 0, n)
    p = 148 * 4 * 256

    def step():
        oracle.reduce_i64(oracle.SUM, xi, p=p)
        oracle.reduce_i64(oracle.MAX, xi, p=p)
        oracle.reduce_f32(oracle.SUM, xf, p=p)
        oracle.reduce_f32(oracle.MAX, xf, p=p)

    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = (time.perf_counter() - t0) / args.steps
    gbs = n * 12 / dt / 1e9
    print(json.dumps({
        "impl": "reference", "metric": C2_METRIC,
        "value": gbs, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3 * (1 << 30) / n, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "i64+f32", "data": "synthetic",
        "config": dict(c2_config(args.sched or "static", world), sample="n=2^24 of the same stream per step"),
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": "2^24 int64 + 2^24 fp32 elements (sum and max each), scaled by bytes"},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def cpu_baseline_reduce():
    import oracle
    import synth
    n = 1 << 26
    xi = synth.c_i64_sym(6, 0, n)
    xf = synth.c_f32_unit(7, 0, n)
    p = 148 * 4 * 256
    t0 = time.perf_counter()
    oracle.reduce_i64(oracle.SUM, xi, p=p)
    oracle.reduce_i64(oracle.MAX, xi, p=p)
    oracle.reduce_f32(oracle.SUM, xf, p=p)
    oracle.reduce_f32(oracle.MAX, xf, p=p)
    dt = time.perf_counter() - t0
    return {"value": n * 12 / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": "2^26 int64 + 2^26 fp32 elements, sum and max each (one pass per op), "
                      "GB/s counted as 12 B per element pair like the GPU metric"}


def cpu_baseline_jacobi():
    import oracle
    import synth
    ny = nx = 2048
    S = 10
    g = synth.jacobi_init(ny, nx)
    t0 = time.perf_counter()
    oracle.jacobi5(g, S)
    dt = time.perf_counter() - t0
    return {"value": (ny - 2) * (nx - 2) * S / dt / 1e9, "unit": "GLUP/s", "cores": 1, "kind": "oracle",
            "sample": "2048^2 grid, 10 sweeps (fp64 oracle), GLUP/s"}


# --------------------------------------------------------------------------- UPIR arm
def pin_to_gpu_numa(local):
    """Run on the CPU cores local to this GPU, so pinned host buffers (first
    touch) land on the GPU's NUMA node: the e2e H2D then runs at PCIe line
    rate instead of crossing the socket interconnect."""
    try:
        import pynvml
        import torch
        pynvml.nvmlInit()
        pr = torch.cuda.get_device_properties(local)
        bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
        h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= set(range(os.cpu_count() or 1))
        if cpus:
            os.sched_setaffinity(0, cpus)
            return len(cpus)
    except Exception:
        pass
    return None


def run_upir(args):
    import torch
    import paper_2209_10643_b200 as U

    rank, world, local = dist_env()
    # test hook (not a bench configuration): every rank on cuda:0, gloo for
    # the host plumbing, a communicator-less upir world (peer windows only) --
    # exercises the N > 1 code of this script on a one-GPU box
    shared = os.environ.get("UPIR_BENCH_SHARED_GPU") == "1"
    if shared:
        local = 0
        os.environ["LOCAL_RANK"] = "0"
    torch.cuda.set_device(local)
    numa_cpus = pin_to_gpu_numa(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
        _PG[0] = dist
        if shared:
            ctx = U.upir_init(local, rank=rank, nranks=world, nccl_id=None)
        else:
            idb = [U.upir_comm_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(idb, src=0)
            ctx = U.upir_init(local, rank=rank, nranks=world, nccl_id=idb[0])
    else:
        ctx = U.upir_init(local)
    stream = torch.cuda.ExternalStream(U.upir_ctx_stream(ctx, 0))
    peaks, peak_src = measured_peaks()

    def barrier():
        U.upir_sync(ctx)
        if pg:
            pg.barrier()
        torch.cuda.synchronize()

    if args.workload == "reduce":
        res = bench_reduce(args, U, ctx, stream, barrier, rank, world, peaks, peak_src)
    elif args.workload == "reduce34":
        res = bench_reduce34(args, U, ctx, stream, barrier, rank, world, peaks, peak_src)
    elif args.workload == "jacobi32k":
        res = bench_jacobi32k(args, U, ctx, stream, barrier, rank, world, peaks, peak_src)
    else:
        raise SystemExit(f"workload {args.workload} is a kernel line of the default run (see 'kernels')")
    # the other loop bodies of the path, each timed on its own (single GPU)
    if world == 1 and not args.no_kernels and args.workload == "reduce":
        res["kernels"] = {}
        # the tensor-core matmuls last: they drive the board into its power cap
        # (sw_power_cap), which would otherwise throttle the ALU-bound stencil
        for name, fn in (("axpy", bench_axpy), ("jacobi", bench_jacobi), ("matvec", bench_matvec),
                         ("stencil7", bench_stencil7), ("matmul", bench_matmul)):
            try:
                res["kernels"][name] = fn(args, U, ctx, stream, peaks, peak_src)
            except Exception as e:   # report, never hide
                res["kernels"][name] = {"error": str(e)[:300]}
    # max over ranks of the timed values
    if args.workload == "reduce":
        if pg:
            t = torch.tensor([res["ms_per_step"], res["e2e_ms"]], device="cuda")
            pg.all_reduce(t, op=pg.ReduceOp.MAX)
            res["ms_per_step"], res["e2e_ms"] = t.tolist()
        res["value"] = res["bytes_all_ranks"] / (res["ms_per_step"] / 1e3) / 1e9
        res["e2e"]["value"] = res["bytes_all_ranks"] / (res["e2e_ms"] / 1e3) / 1e9
    elif args.workload == "reduce34":
        res["value"] = res["bytes_all_ranks"] / (res["ms_per_step"] / 1e3) / 1e9
    else:
        res["value"] = res.pop("glups")
    if rank == 0:
        out = {k: v for k, v in res.items() if k not in ("bytes_all_ranks", "e2e_ms")}
        if isinstance(out.get("e2e"), dict):
            out["e2e"]["host_affinity_cpus"] = numa_cpus
        if world == 1 and not args.no_cpu_baseline:
            out["cpu_baseline"] = cpu_baseline_jacobi() if args.workload == "jacobi32k" else cpu_baseline_reduce()
        print(json.dumps(out), flush=True)
    U.upir_finalize(ctx)
    if pg:
        pg.destroy_process_group()


def bench_reduce(args, U, ctx, stream, barrier, rank, world, peaks, peak_src):
    import torch
    n = 1 << args.n_log2
    teams, units = 148 * 4, 256
    # static1 / dynamic: chunk = one 16-B vector per unit (2 int64 / 4 fp32)
    pol = {"static": U.SCHED_STATIC, "static1": U.SCHED_STATIC, "dynamic": U.SCHED_DYNAMIC}[args.sched]
    ci, cf = (0, 0) if args.sched == "static" else (2, 4)
    # device-resident inputs: map(alloc) + on-device synthetic fill (rank r
    # holds global elements [r*n, (r+1)*n) of each stream)
    hi = np.empty(1, np.int64)          # host key objects for the alloc maps
    hf = np.empty(1, np.float32)
    xi_t = torch.empty(n, dtype=torch.int64, device="cuda")
    xf_t = torch.empty(n, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    mi = U.upir_data_adopt(ctx, xi_t)
    mf = U.upir_data_adopt(ctx, xf_t)
    U.upir_synth_fill(ctx, mi, 2, 6, rank * n)
    U.upir_synth_fill(ctx, mf, 0, 7, rank * n)
    res_t = torch.zeros(8, dtype=torch.float64, device="cuda")   # 4 local + 4 world results (8 B each)
    torch.cuda.synchronize()
    base = res_t.data_ptr()
    reds_i = [U.reduction(U.OP_SUM, U.I64, base + 0), U.reduction(U.OP_MAX, U.I64, base + 8)]
    reds_f = [U.reduction(U.OP_SUM, U.F32, base + 16), U.reduction(U.OP_MAX, U.F32, base + 24)]
    peer = use_peer(world)
    if peer:
        U.upir_peer_share(ctx)
    wflag = U.WORLD_REDUCE if peer else 0
    loop_i = U.loop_desc(0, n, policy=pol, chunk=ci, flags=wflag)
    loop_f = U.loop_desc(0, n, policy=pol, chunk=cf, flags=wflag)
    spmd = U.upir_spmd_launch(ctx, U.spmd_desc(teams, units))
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]

    def step(timed_events=None):
        e = timed_events
        if e:
            e[0].record(stream)
        U.upir_loop_exec(spmd, loop_i, U.body(U.BODY_REDUCE, U.I64, in0=mi), reds_i)
        if e:
            e[1].record(stream)
        U.upir_loop_exec(spmd, loop_f, U.body(U.BODY_REDUCE, U.F32, in0=mf), reds_f)
        if e:
            e[2].record(stream)
        if world > 1 and not peer:
            U.upir_reduce(ctx, U.OP_SUM, U.I64, base + 0, 1, base + 32, U.SCOPE_WORLD)
            U.upir_reduce(ctx, U.OP_MAX, U.I64, base + 8, 1, base + 40, U.SCOPE_WORLD)
            U.upir_reduce(ctx, U.OP_SUM, U.F32, base + 16, 1, base + 48, U.SCOPE_WORLD)
            U.upir_reduce(ctx, U.OP_MAX, U.F32, base + 24, 1, base + 56, U.SCOPE_WORLD)

    for _ in range(args.warmup):
        step()
    barrier()
    st0 = U.upir_ctx_stats(ctx)["launches"]
    clk = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clk.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for k in range(args.steps):
        step(evs[k])
    t1.record(stream)
    barrier()
    k_i = [e[0].elapsed_time(e[1]) for e in evs]
    k_f = [e[1].elapsed_time(e[2]) for e in evs]
    clocks = clk.stop()
    launches = U.upir_ctx_stats(ctx)["launches"] - st0
    ms = t0.elapsed_time(t1) / args.steps
    # correctness guard on the last step (cheap properties)
    r = res_t.cpu()
    assert -(1 << 28) <= r[1:2].view(torch.int64).item() < (1 << 28)
    U.upir_spmd_end(spmd)

    # ---- e2e: host buffers through the C-ABI ------------------------------------
    import ctypes
    e2e_n = n if args.e2e_steps > 0 else 1
    hx_i = torch.empty(e2e_n, dtype=torch.int64, pin_memory=True)
    hx_f = torch.empty(e2e_n, dtype=torch.float32, pin_memory=True)
    hx_i.copy_(xi_t[:e2e_n])
    hx_f.copy_(xf_t[:e2e_n])
    # result scalars: a pinned host buffer (no per-step page registration)
    hres_t = torch.zeros(8, dtype=torch.float64, pin_memory=True)
    hres = np.ctypeslib.as_array(ctypes.cast(hres_t.data_ptr(), ctypes.POINTER(ctypes.c_double)), shape=(8,))
    U.upir_data_unmap(ctx, mi)
    U.upir_data_unmap(ctx, mf)
    del xi_t, xf_t
    torch.cuda.synchronize()
    torch.cuda.empty_cache()

    def host_arr(t):
        return np.ctypeslib.as_array(ctypes.cast(t.data_ptr(), ctypes.POINTER(
            ctypes.c_int64 if t.dtype == torch.int64 else ctypes.c_float)), shape=(t.numel(),))

    ai, af = host_arr(hx_i), host_arr(hx_f)

    def e2e_step():
        m1 = U.upir_data_map(ctx, ai, U.MAP_TO)
        m2 = U.upir_data_map(ctx, af, U.MAP_TO)
        mr = U.upir_data_map(ctx, hres, U.MAP_FROM)
        rp, _, _ = U.upir_data_device_ptr(mr)
        s = U.upir_spmd_launch(ctx, U.spmd_desc(teams, units))
        U.upir_loop_exec(s, U.loop_desc(0, e2e_n, policy=pol, chunk=ci, flags=wflag),
                         U.body(U.BODY_REDUCE, U.I64, in0=m1),
                         [U.reduction(U.OP_SUM, U.I64, rp + 0), U.reduction(U.OP_MAX, U.I64, rp + 8)])
        U.upir_loop_exec(s, U.loop_desc(0, e2e_n, policy=pol, chunk=cf, flags=wflag),
                         U.body(U.BODY_REDUCE, U.F32, in0=m2),
                         [U.reduction(U.OP_SUM, U.F32, rp + 16), U.reduction(U.OP_MAX, U.F32, rp + 24)])
        if world > 1 and not peer:
            for k, (op, dt) in enumerate(((U.OP_SUM, U.I64), (U.OP_MAX, U.I64), (U.OP_SUM, U.F32),
                                          (U.OP_MAX, U.F32))):
                U.upir_reduce(ctx, op, dt, rp + 8 * k, 1, rp + 32 + 8 * k, U.SCOPE_WORLD)
        U.upir_spmd_end(s)
        U.upir_data_unmap(ctx, mr)
        U.upir_data_unmap(ctx, m2)
        U.upir_data_unmap(ctx, m1)
        U.upir_sync(ctx)

    e2e_ms = float("nan")
    if args.e2e_steps > 0:
        e2e_step()   # warm-up (pins the host ranges once)
        barrier()
        te0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        barrier()
        e2e_ms = (time.perf_counter() - te0) * 1e3 / args.e2e_steps
        if os.environ.get("UPIR_E2E_PHASES"):
            tp = time.perf_counter()
            m1 = U.upir_data_map(ctx, ai, U.MAP_TO)
            U.upir_sync(ctx)
            t_map = time.perf_counter() - tp
            U.upir_data_unmap(ctx, m1)
            U.upir_sync(ctx)
            print(f"e2e phase: map(to) of {ai.nbytes / 1e9:.2f} GB in {t_map * 1e3:.1f} ms "
                  f"= {ai.nbytes / t_map / 1e9:.1f} GB/s", file=sys.stderr)
    # the e2e path is timed by the host clock around synchronous steps (each
    # step ends in upir_sync), max over ranks below

    bytes_rank = n * 8 + n * 4
    ki, kf = statistics.mean(k_i), statistics.mean(k_f)
    ach_i = n * 8 / (ki / 1e3) / 1e9
    ach_f = n * 4 / (kf / 1e3) / 1e9
    peak = float(peaks["hbm_gbs"])
    return {
        "metric": C2_METRIC,
        "value": None, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "i64+f32", "data": "synthetic",
        "config": dict(c2_config(args.sched, world), n_per_gpu=n),
        "roofline": {"bound": "hbm", "achieved": ach_i, "peak": peak, "unit": "GB/s",
                     "frac": ach_i / peak, "traffic": ncu_traffic("reduce_i64"),
                     "kernel": "stream_loop_kernel<RED_I64,2>", "peak_source": peak_src,
                     "other_kernels": {"reduce_f32": {"achieved": ach_f, "frac": ach_f / peak,
                                                      "traffic": ncu_traffic("reduce_f32")}}},
        "kernel_ms": {"reduce_i64": ki, "reduce_f32": kf},
        "clocks": clocks,
        "gpu_launches": launches,
        "e2e": {"value": None, "unit": "GB/s", "h2d_bytes_per_step": bytes_rank, "d2h_bytes_per_step": 32},
        "bytes_all_ranks": bytes_rank * world, "e2e_ms": e2e_ms,
    }


def _time_graph(U, ctx, stream, launch, reps):
    import torch
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    U.upir_sync(ctx)
    e0.record(stream)
    for _ in range(reps):
        launch()
    e1.record(stream)
    U.upir_sync(ctx)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def bench_axpy(args, U, ctx, stream, peaks, peak_src):
    """a6 axpy y = y + a*x with a fused fp32 sum (C1 body) at n = 2^28."""
    import torch
    n = 1 << 28
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    r = torch.zeros(1, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    mx, my = U.upir_data_adopt(ctx, x), U.upir_data_adopt(ctx, y)
    U.upir_synth_fill(ctx, mx, 0, 1)
    U.upir_synth_fill(ctx, my, 0, 2)
    out = {}
    s = U.upir_spmd_launch(ctx, U.spmd_desc(148 * 4, 256))
    for label, pol, c in (("static", U.SCHED_STATIC, 0), ("static4", U.SCHED_STATIC, 4)):
        loop = U.loop_desc(0, n, policy=pol, chunk=c)
        body = U.body(U.BODY_AXPY, U.F32, in0=mx, out=my, alpha=2.0)
        red = [U.reduction(U.OP_SUM, U.F32, r)]
        for _ in range(3):
            U.upir_loop_exec(s, loop, body, red)
        ms = _time_graph(U, ctx, stream, lambda: U.upir_loop_exec(s, loop, body, red), 10)
        gbs = 12 * n / (ms / 1e3) / 1e9
        out[label] = {"ms": ms, "GB/s": gbs, "frac": gbs / float(peaks["hbm_gbs"])}
    U.upir_spmd_end(s)
    U.upir_data_unmap(ctx, mx)
    U.upir_data_unmap(ctx, my)
    U.upir_sync(ctx)
    return {"workload": "axpy y=y+2x + fused fp32 sum, n=2^28, 592x256, 12 B/iter", "peak_source": peak_src,
            "bound": "hbm", **out}


def jacobi_tile_sched():
    """Tile-loop schedule of the Jacobi lines: (chunk, tile order); chunk 0 =
    static block, 'col' = UPIR_TILE_COLMAJOR (reading c35).  Env overrides
    UPIR_JACOBI_CHUNK / UPIR_JACOBI_ORDER are sweep hooks."""
    return int(os.environ.get("UPIR_JACOBI_CHUNK", 1)), os.environ.get("UPIR_JACOBI_ORDER", "row")


def bench_jacobi(args, U, ctx, stream, peaks, peak_src, ny=8192, nx=8192, S=100):
    """C3: 2-D Jacobi 5-point 8192^2 fp32, 100 sweeps as one CUDA graph, tiles
    32x256 static,1 over 296 teams, intra-tile static,4 over 256 units."""
    import torch
    a_t = torch.empty(ny * nx, dtype=torch.float32, device="cuda")
    b_t = torch.empty(ny * nx, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    ma, mb = U.upir_data_adopt(ctx, a_t), U.upir_data_adopt(ctx, b_t)
    U.upir_synth_fill(ctx, ma, 4, 5, 0, ny, nx)
    U.upir_synth_fill(ctx, mb, 4, 5, 0, ny, nx)
    # 16x256 tiles, 3 teams per SM: measured best of the r01 sweep (tools/sweep_jacobi_axpy.sh)
    teams = int(os.environ.get("UPIR_JACOBI_TEAMS", 444))
    bm, bn = (int(v) for v in os.environ.get("UPIR_JACOBI_TILE", "16x256").split("x"))
    chunk, order = jacobi_tile_sched()
    loop = U.loop_desc([1, 1], [ny - 1, nx - 1], tile=[bm, bn], policy=U.SCHED_STATIC, chunk=chunk,
                       distribute=U.DIST_TEAMS, inner_chunk=4, flags=U.TILE_COLMAJOR if order == "col" else 0)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(teams, 256))
    bodies = [U.body(U.BODY_JACOBI5, U.F32, in0=ma, out=mb, ld=(nx, 0, 0), dims=(ny, 0, 0)),
              U.body(U.BODY_JACOBI5, U.F32, in0=mb, out=ma, ld=(nx, 0, 0), dims=(ny, 0, 0))]
    U.upir_graph_begin(ctx)
    for k in range(S):
        U.upir_loop_exec(s, loop, bodies[k % 2])
    g = U.upir_graph_end(ctx)
    for _ in range(2):
        U.upir_graph_launch(ctx, g)
    reps = max(2, min(args.steps, 5))
    ms = _time_graph(U, ctx, stream, lambda: U.upir_graph_launch(ctx, g), reps)
    lups = (ny - 2) * (nx - 2) * S
    glups = lups / (ms / 1e3) / 1e9
    gbs = 8 * lups / (ms / 1e3) / 1e9
    U.upir_graph_destroy(g)
    U.upir_spmd_end(s)
    U.upir_data_unmap(ctx, ma)
    U.upir_data_unmap(ctx, mb)
    U.upir_sync(ctx)
    peak = float(peaks["hbm_gbs"])
    return {"workload": f"C3: Jacobi 5-point {ny}x{nx} fp32, {S} sweeps (one CUDA graph), tiles {bm}x{bn} "
                        f"static,1 over {teams} teams, static,4 over 256 units",
            "ms_per_100_sweeps": ms, "GLUP/s": glups, "bound": "hbm",
            "roofline": {"achieved": gbs, "peak": peak, "unit": "GB/s", "frac": gbs / peak,
                         "algorithmic_bytes_per_lup": 8, "peak_source": peak_src,
                         "traffic": ncu_traffic("jacobi")}}


def bench_stencil7(args, U, ctx, stream, peaks, peak_src):
    """NEXT #4: 2-D filter stencil, filter size 7 (the paper's stencil,
    PAPER.md:1483), at the paper's largest size 2048^2 and at 8192^2."""
    import torch
    out = {}
    v = torch.tensor([1, 2, 3, 4, 3, 2, 1], dtype=torch.float64)
    w = (torch.outer(v, v) / 256.0).float().cuda()
    for n in (2048, 8192):
        a_t = torch.empty(n * n, dtype=torch.float32, device="cuda")
        b_t = torch.empty(n * n, dtype=torch.float32, device="cuda")
        torch.cuda.synchronize()
        ma, mb, mw = U.upir_data_adopt(ctx, a_t), U.upir_data_adopt(ctx, b_t), U.upir_data_adopt(ctx, w)
        U.upir_synth_fill(ctx, ma, 4, 5, 0, n, n)
        U.upir_synth_fill(ctx, mb, 4, 5, 0, n, n)
        lups = (n - 6) ** 2
        cfgs = ((444, 128, (8, 512)), (592, 256, (16, 128)), (296, 128, (16, 512)), (888, 64, (8, 256)))
        if os.environ.get("UPIR_STENCIL_CFGS"):   # sweep hook: "TEAMSxUNITS:BMxBN,..."
            cfgs = [tuple(int(x) for x in g.split(":")[0].split("x")) + (tuple(int(x) for x in g.split(":")[1].split("x")),)
                    for g in os.environ["UPIR_STENCIL_CFGS"].split(",")]
        for teams, units, tile in cfgs:
            s = U.upir_spmd_launch(ctx, U.spmd_desc(teams, units))
            loop = U.loop_desc([3, 3], [n - 3, n - 3], tile=list(tile), chunk=1, distribute=U.DIST_TEAMS,
                               inner_chunk=4)
            body = U.body(U.BODY_STENCIL2D, U.F32, in0=ma, in1=mw, out=mb, ld=(n, 0, 0), dims=(n, 7, 0))
            for _ in range(3):
                U.upir_loop_exec(s, loop, body)
            ms = _time_graph(U, ctx, stream, lambda: U.upir_loop_exec(s, loop, body), 10)
            U.upir_spmd_end(s)
            out[f"{n}x{n} tile {tile[0]}x{tile[1]} {teams}x{units}"] = {
                "ms_per_sweep": ms, "GLUP/s": lups / (ms / 1e3) / 1e9, "GB/s": 8 * lups / (ms / 1e3) / 1e9,
                "GFLOP/s": 98 * lups / (ms / 1e3) / 1e9}
        for m in (mw, mb, ma):
            U.upir_data_unmap(ctx, m)
        U.upir_sync(ctx)
        del a_t, b_t
    fp32_peak = 72.5   # TFLOP/s: measured FFMA rate on this B200 (tools/debug/ffma_rate.cu)
    best = max(v["GFLOP/s"] for k, v in out.items() if k.startswith("8192"))
    return {"workload": "2-D 7x7 filter stencil (49 taps, fp32 FMA), tile loop static,1 over the teams, "
                        "static,4 over the units (BN = 4 x units: one 4-column strip per unit); one sweep per launch",
            "bound": "alu (49 FMA per point)",
            "roofline": {"bound": "alu", "achieved": best / 1e3, "peak": fp32_peak, "unit": "TFLOP/s",
                         "frac": best / 1e3 / fp32_peak, "peak_source": "measured FFMA microbenchmark"},
            "paper_v100_end_to_end_ms_2048": 56.47, **out}


def bench_matvec(args, U, ctx, stream, peaks, peak_src, n=16384):
    """NEXT #2: matvec y = A x at the paper's largest size N = 16384
    (PAPER.md:1430), rows static,1 over 592 teams, k static,4 over 256 units."""
    import torch
    A = torch.empty(n * n, dtype=torch.float32, device="cuda")
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    ma, mx, my = U.upir_data_adopt(ctx, A), U.upir_data_adopt(ctx, x), U.upir_data_adopt(ctx, y)
    U.upir_synth_fill(ctx, ma, 1, 3)
    U.upir_synth_fill(ctx, mx, 1, 1)
    out = {}
    for teams, units in ((592, 256), (296, 512)):
        s = U.upir_spmd_launch(ctx, U.spmd_desc(teams, units))
        loop = U.loop_desc(0, n, chunk=1, distribute=U.DIST_TEAMS, inner_chunk=4)
        body = U.body(U.BODY_MATVEC, U.F32, in0=ma, in1=mx, out=my, ld=(n, 0, 0), dims=(n, n, 0))
        for _ in range(3):
            U.upir_loop_exec(s, loop, body)
        ms = _time_graph(U, ctx, stream, lambda: U.upir_loop_exec(s, loop, body), 10)
        U.upir_spmd_end(s)
        gbs = 4.0 * n * n / (ms / 1e3) / 1e9
        out[f"{teams}x{units}"] = {"ms": ms, "GB/s": gbs, "frac": gbs / float(peaks["hbm_gbs"])}
    for m in (my, mx, ma):
        U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)
    del A
    return {"workload": f"matvec {n}x{n} fp32 (PAPER.md:1430 size), rows static,1 over teams, "
                        "k static,4 over units + reduction(+); 4 B of A per iteration", "bound": "hbm",
            "peak_source": peak_src, "paper_v100_end_to_end_ms": 583.45, **out}


def bench_matmul(args, U, ctx, stream, peaks, peak_src, n=8192):
    """C4: dense bf16 matmul 8192^3 -> fp32 as a collapse(2) upir.loop, 128x256
    output tiles static,1 over 148 persistent teams (tcgen05 path)."""
    import torch
    A = torch.empty(n * n, dtype=torch.bfloat16, device="cuda")
    B = torch.empty(n * n, dtype=torch.bfloat16, device="cuda")
    C = torch.empty(n * n, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    ma, mb, mc = U.upir_data_adopt(ctx, A), U.upir_data_adopt(ctx, B), U.upir_data_adopt(ctx, C)
    U.upir_synth_fill(ctx, ma, 3, 3)
    U.upir_synth_fill(ctx, mb, 3, 4)
    teams = int(os.environ.get("UPIR_MATMUL_TEAMS", 148))
    s = U.upir_spmd_launch(ctx, U.spmd_desc(teams, 256))
    loop = U.loop_desc([0, 0], [n, n], policy=U.SCHED_STATIC, chunk=1, distribute=U.DIST_TEAMS)
    body = U.body(U.BODY_MATMUL, U.BF16, in0=ma, in1=mb, out=mc, ld=(n, n, n), dims=(n, n, n))
    for _ in range(3):
        U.upir_loop_exec(s, loop, body)
    reps = max(3, min(args.steps, 10))
    ms = _time_graph(U, ctx, stream, lambda: U.upir_loop_exec(s, loop, body), reps)
    U.upir_spmd_end(s)
    for m in (mc, mb, ma):
        U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)
    del A, B
    tflops = 2.0 * n ** 3 / (ms / 1e3) / 1e12
    peak = float(peaks.get("bf16_tflops", 1590.0))
    # CTA pairs (cta_group::2): 74 teams of 2 CTAs = 512 units, 256 x 256 tiles
    pair = {}
    A2 = torch.empty(n * n, dtype=torch.bfloat16, device="cuda")
    B2 = torch.empty(n * n, dtype=torch.bfloat16, device="cuda")
    torch.cuda.synchronize()
    ma2, mb2, mc = U.upir_data_adopt(ctx, A2), U.upir_data_adopt(ctx, B2), U.upir_data_adopt(ctx, C)
    U.upir_synth_fill(ctx, ma2, 3, 3)
    U.upir_synth_fill(ctx, mb2, 3, 4)
    try:
        sp = U.upir_spmd_launch(ctx, U.spmd_desc(74, 512))
        bodyp = U.body(U.BODY_MATMUL, U.BF16, in0=ma2, in1=mb2, out=mc, ld=(n, n, n), dims=(n, n, n))
        for _ in range(3):
            U.upir_loop_exec(sp, loop, bodyp)
        msp = _time_graph(U, ctx, stream, lambda: U.upir_loop_exec(sp, loop, bodyp), reps)
        U.upir_spmd_end(sp)
        pair = {"ms": msp, "TFLOP/s": 2.0 * n ** 3 / (msp / 1e3) / 1e12,
                "frac": 2.0 * n ** 3 / (msp / 1e3) / 1e12 / peak,
                "geometry": "74 teams x 512 units (CTA pairs, tcgen05.mma.cta_group::2, 256x256 tiles)"}
    except Exception as e:
        pair = {"error": str(e)[:200]}
    for m in (mc, mb2, ma2):
        U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)
    del A2, B2
    # fp32 inputs (3xTF32 on kind::tf32): 384 units per team
    A32 = torch.empty(n * n, dtype=torch.float32, device="cuda")
    B32 = torch.empty(n * n, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    ma32, mb32, mc = U.upir_data_adopt(ctx, A32), U.upir_data_adopt(ctx, B32), U.upir_data_adopt(ctx, C)
    U.upir_synth_fill(ctx, ma32, 1, 3)
    U.upir_synth_fill(ctx, mb32, 1, 4)
    body32 = U.body(U.BODY_MATMUL, U.F32, in0=ma32, in1=mb32, out=mc, ld=(n, n, n), dims=(n, n, n))
    f32_variants = {}
    for label, tms, uns in (("single_cta", teams, 384), ("cta_pair", 74, 768)):
        s32 = U.upir_spmd_launch(ctx, U.spmd_desc(tms, uns))
        U.upir_loop_exec(s32, loop, body32)
        f32_variants[label] = _time_graph(U, ctx, stream, lambda: U.upir_loop_exec(s32, loop, body32), 3)
        U.upir_spmd_end(s32)
    ms32 = min(f32_variants.values())
    for m in (mc, mb32, ma32):
        U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)
    del A32, B32
    tf32_peak = peak / 2.0      # tf32 dense = 1/2 of bf16 (nominal ratio) x measured bf16
    fp32_tflops = 2.0 * n ** 3 / (ms32 / 1e3) / 1e12
    # headline: the better of the single-CTA and CTA-pair realisations of the
    # same collapse(2) loop (both parity-tested)
    best = pair if pair.get("TFLOP/s", 0) > tflops else {"ms": ms, "TFLOP/s": tflops}
    return {"workload": f"C4: bf16 matmul {n}^3 -> fp32 as a collapse(2) upir.loop, tile loop static,1 over "
                        "persistent teams: 74 teams x 512 units (CTA pairs, tcgen05.mma.cta_group::2, 256x256 tiles) "
                        f"and {teams} teams x 256 units (1 CTA, 128x256 tiles); TMA SW128, TMEM accumulators",
            "ms": best["ms"], "TFLOP/s": best["TFLOP/s"], "bound": "tensor", "cta_pair_bf16": pair,
            "single_cta_bf16": {"ms": ms, "TFLOP/s": tflops, "frac": tflops / peak},
            "fp32_3xtf32": {"ms": ms32, "TFLOP/s": fp32_tflops, "tensor_TFLOP/s": 3 * fp32_tflops,
                            "variants_ms": f32_variants,
                            "peak_tf32": tf32_peak, "frac_of_tf32_over_3": fp32_tflops / (tf32_peak / 3),
                            "peak_source": peak_src + " bf16 burst x nominal tf32/bf16 ratio 1/2"},
            "roofline": {"achieved": best["TFLOP/s"], "peak": peak, "unit": "TFLOP/s", "frac": best["TFLOP/s"] / peak,
                         "peak_source": peak_src + " bf16 burst", "traffic": ncu_traffic("matmul")}}


def _ranks_max(pg, vals):
    import torch
    if not pg:
        return vals
    t = torch.tensor(vals, dtype=torch.float64, device="cuda")
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return t.tolist()


def bench_reduce34(args, U, ctx, stream, barrier, rank, world, peaks, peak_src):
    """C5a: one int64 sum+max reduction over n = 2^34 elements distributed over
    the ranks (upir_dist BLOCK, CLUSTER-target loop), combined with
    upir_reduce(WORLD).  Strong scaling (the global n is fixed)."""
    import torch
    n = 1 << int(os.environ.get("UPIR_C5A_LOG2", 34))
    lo, hi = U.upir_dist_owned_rows(n, rank, world)
    x = torch.empty(hi - lo, dtype=torch.int64, device="cuda")
    res_t = torch.zeros(4, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    m = U.upir_data_adopt(ctx, x, U.dist(n, 1, 8))
    U.upir_synth_fill(ctx, m, 2, 6)
    base = res_t.data_ptr()
    reds = [U.reduction(U.OP_SUM, U.I64, base), U.reduction(U.OP_MAX, U.I64, base + 8)]
    spmd = U.upir_spmd_launch(ctx, U.spmd_desc(148 * 4, 256, U.TARGET_CLUSTER))
    pol = {"static": U.SCHED_STATIC, "static1": U.SCHED_STATIC, "dynamic": U.SCHED_DYNAMIC}[args.sched]
    peer = use_peer(world)
    if peer:
        U.upir_peer_share(ctx)
    loop = U.loop_desc(0, n, policy=pol, chunk=0 if args.sched == "static" else 2,
                       flags=U.WORLD_REDUCE if world > 1 else 0)

    def step():
        # world > 1: the allreduce is part of the loop (in-kernel over peer
        # windows, or upir_reduce(WORLD) after it with UPIR_PEER=0)
        U.upir_loop_exec(spmd, loop, U.body(U.BODY_REDUCE, U.I64, in0=m), reds)

    for _ in range(args.warmup):
        step()
    barrier()
    st0 = U.upir_ctx_stats(ctx)["launches"]
    clk = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clk.start()
    ms = _time_graph(U, ctx, stream, step, args.steps)
    barrier()
    clocks = clk.stop()
    launches = U.upir_ctx_stats(ctx)["launches"] - st0
    ms_local = ms
    (ms,) = _ranks_max(pg_of(), [ms])
    U.upir_spmd_end(spmd)
    U.upir_data_unmap(ctx, m)
    U.upir_sync(ctx)
    peak = float(peaks["hbm_gbs"])
    per_rank_gbs = (hi - lo) * 8 / (ms_local / 1e3) / 1e9
    return {
        "metric": "GB/s of the 2^34-element int64 sum+max reduction (C5a), whole job", "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "i64", "data": "synthetic",
        "config": {"workload": f"C5a: int64 sum+max over n=2^{int(math.log2(n))} BLOCK-distributed over {world} "
                               f"GPU(s), 592x256 per GPU, schedule {args.sched}, "
                               f"world reduction {'fused in-kernel (peer windows)' if peer else 'NCCL'}",
                   "n_global": n, "parallelism": f"dp{world}", "l2": "inputs >> L2"},
        "roofline": {"bound": "hbm", "achieved": per_rank_gbs, "peak": peak, "unit": "GB/s",
                     "frac": per_rank_gbs / peak, "traffic": ncu_traffic("reduce_i64_1"),
                     "kernel": "stream_loop_kernel<RED_I64,1 or 2> (per rank)", "peak_source": peak_src},
        "clocks": clocks, "gpu_launches": launches,
        "e2e": {"value": None, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "note": "inputs generated on device (2^34 x 8 B exceeds host staging)"},
        "bytes_all_ranks": n * 8, "e2e_ms": float("nan"),
    }


_PG = [None]


_PEER_OK = [None]


def use_peer(world):
    """N > 1: exchange through NVLink peer windows (fused world reduction /
    fused halo) unless UPIR_PEER=0 selects the NCCL path, or some rank's GPU
    cannot map another's memory (decided collectively, so all ranks agree)."""
    if world == 1 or os.environ.get("UPIR_PEER", "1") == "0":
        return False
    if _PEER_OK[0] is None:
        import torch
        me = torch.cuda.current_device()
        ok = all(torch.cuda.can_device_access_peer(me, d) for d in range(torch.cuda.device_count()) if d != me)
        t = torch.tensor([1 if ok else 0], dtype=torch.int32)
        if os.environ.get("UPIR_BENCH_SHARED_GPU") != "1":
            t = t.cuda()
        _PG[0].all_reduce(t, op=_PG[0].ReduceOp.MIN)
        _PEER_OK[0] = bool(t.item())
    return _PEER_OK[0]


def pg_of():
    return _PG[0]


def bench_jacobi32k(args, U, ctx, stream, barrier, rank, world, peaks, peak_src, n=None, S=100):
    """C5b: Jacobi 5-point on a 32768^2 fp32 grid, 100 sweeps, BLOCK row slabs
    with 1-row halos exchanged by upir_sync(HALO) before every sweep (NCCL
    send/recv in stream order), the 100 sweeps captured as one CUDA graph.
    Strong scaling."""
    import torch
    n = n or int(os.environ.get("UPIR_C5B_N", 32768))
    lo, hi = U.upir_dist_owned_rows(n, rank, world)
    llo, lhi = max(0, lo - 1), min(n, hi + 1)
    a_t = torch.empty((lhi - llo) * n, dtype=torch.float32, device="cuda")
    b_t = torch.empty((lhi - llo) * n, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    d = U.dist(n, n, 4, halo_rows=1)
    ma, mb = U.upir_data_adopt(ctx, a_t, d), U.upir_data_adopt(ctx, b_t, d)
    U.upir_synth_fill(ctx, ma, 4, 5, 0, n, n)
    U.upir_synth_fill(ctx, mb, 4, 5, 0, n, n)
    peer = use_peer(world)
    if peer:   # fused halo: boundary rows stored into the neighbours' halos inside each sweep
        U.upir_peer_share(ctx, [ma, mb])
    teams = int(os.environ.get("UPIR_JACOBI_TEAMS", 444))
    bm, bn = (int(v) for v in os.environ.get("UPIR_JACOBI_TILE", "16x256").split("x"))
    chunk, order = jacobi_tile_sched()
    loop = U.loop_desc([1, 1], [n - 1, n - 1], tile=[bm, bn], policy=U.SCHED_STATIC, chunk=chunk,
                       distribute=U.DIST_TEAMS, inner_chunk=4, flags=U.TILE_COLMAJOR if order == "col" else 0)
    s = U.upir_spmd_launch(ctx, U.spmd_desc(teams, 256, U.TARGET_CLUSTER))
    bodies = [(ma, U.body(U.BODY_JACOBI5, U.F32, in0=ma, out=mb, ld=(n, 0, 0), dims=(n, 0, 0))),
              (mb, U.body(U.BODY_JACOBI5, U.F32, in0=mb, out=ma, ld=(n, 0, 0), dims=(n, 0, 0)))]

    def sweeps():
        for k in range(S):
            src, body = bodies[k % 2]
            if not peer:
                U.upir_sync(ctx, U.SYNC_HALO, halo_map=src)
            U.upir_loop_exec(s, loop, body)

    U.upir_graph_begin(ctx)
    sweeps()
    g = U.upir_graph_end(ctx)
    U.upir_graph_launch(ctx, g)
    barrier()
    st0 = U.upir_ctx_stats(ctx)["launches"]
    clk = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
    clk.start()
    reps = max(1, min(args.steps, 3))
    ms_local = _time_graph(U, ctx, stream, lambda: U.upir_graph_launch(ctx, g), reps)
    barrier()
    clocks = clk.stop()
    launches = U.upir_ctx_stats(ctx)["launches"] - st0
    (ms,) = _ranks_max(pg_of(), [ms_local])
    U.upir_graph_destroy(g)
    U.upir_spmd_end(s)
    U.upir_data_unmap(ctx, ma)
    U.upir_data_unmap(ctx, mb)
    U.upir_sync(ctx)
    lups = (n - 2) * (n - 2) * S
    own = (min(hi, n - 1) - max(lo, 1)) * (n - 2) * S
    per_rank_gbs = 8 * own / (ms_local / 1e3) / 1e9
    peak = float(peaks["hbm_gbs"])
    glups = lups / (ms / 1e3) / 1e9
    return {
        "metric": "Jacobi GLUP/s (C5b 32768^2, 100 sweeps), whole job", "unit": "GLUP/s",
        "n_gpus": world, "steps": reps, "warmup": 1, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"C5b: Jacobi 5-point {n}x{n} fp32, {S} sweeps as one CUDA graph, BLOCK row slabs "
                               f"over {world} GPU(s) with 1-row halos "
                               f"({'fused peer stores in each sweep' if peer else 'upir_sync HALO before each sweep'}), tiles "
                               f"{bm}x{bn} static,1 over {teams} teams",
                   "parallelism": f"dp{world}", "l2": "2 x 4 GiB grids >> L2"},
        "roofline": {"bound": "hbm", "achieved": per_rank_gbs, "peak": peak, "unit": "GB/s",
                     "frac": per_rank_gbs / peak, "traffic": ncu_traffic("jacobi32k"),
                     "kernel": f"jacobi5_kernel<{bm},{bn}>", "peak_source": peak_src},
        "clocks": clocks, "gpu_launches": launches,
        "e2e": {"value": None, "unit": "GLUP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "glups": glups, "e2e_ms": float("nan"), "bytes_all_ranks": None,
    }


def main():
    args = parse()
    if args.sched is None:
        args.sched = "static1" if args.workload == "reduce34" else "static"
    if args.impl == "reference":
        run_reference(args)
        return
    run_upir(args)


if __name__ == "__main__":
    main()
