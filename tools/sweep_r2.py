"""Round-2 sweeps on one GPU (experiment driver, not a bench line):
AXPY static-block occupancy / load variants, Jacobi tile orders and chunks
for C3 and C5b.  Env hooks are read by the runtime at every upir_loop_exec,
so one process sweeps them.

    python tools/sweep_r2.py axpy|jacobi|c5b ...
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def args_ns(steps=5):
    return argparse.Namespace(gpus=1, steps=steps, warmup=3, impl="upir", sched="static", n_log2=30, e2e_steps=0,
                              no_cpu_baseline=True, no_kernels=False, no_scaling=False, lines=None)


def setenv(**kv):
    for k, v in kv.items():
        if v is None:
            os.environ.pop(k, None)
        else:
            os.environ[k] = str(v)


def main():
    what = sys.argv[1:]
    E = bench.Env(args_ns())
    out = []
    if "axpy" in what:
        for lb in (None, 0):
            for occ in (None, 1):
                for dvar in (None, 1, 4, 7, 9):
                    setenv(UPIR_DIRECT_OCC=occ, UPIR_DVAR=dvar, UPIR_LB256=lb)
                    r = bench.bench_axpy(E)
                    out.append({"axpy": {"lb256": lb, "occ": occ, "dvar": dvar, **r["summary"]}})
                    print(json.dumps(out[-1]), flush=True)
        setenv(UPIR_DIRECT_OCC=None, UPIR_DVAR=None, UPIR_LB256=None)
    if "reduce" in what:
        for lb in (None, 1):
            setenv(UPIR_LB256=lb)
            r = bench.bench_c2(E)
            out.append({"reduce": {"lb256": lb, **r["summary"]}})
            print(json.dumps(out[-1]), flush=True)
            E.free()
        setenv(UPIR_LB256=None)
    for key, fn in (("jacobi", bench.bench_jacobi), ("c5b", bench.line_c5b)):
        if key not in what:
            continue
        cfgs = [("static", None, c) for c in (1, 8, 16, 32, 37, 64)] + [("dynamic", None, c) for c in (1,)]
        for pol, skew, chunk in cfgs:
            order = "row"
            for teams in (444,):
                setenv(UPIR_JACOBI_ORDER=order, UPIR_JACOBI_CHUNK=chunk, UPIR_JACOBI_TEAMS=teams,
                       UPIR_JACOBI_POLICY=pol)
                try:
                    r = fn(E)
                    summ = r.get("summary") or {k: v for k, v in r["paths"].items()}
                except Exception as e:
                    summ = {"error": str(e)[:200]}
                out.append({key: {"policy": pol, "skew": skew, "chunk": chunk, "teams": teams, **summ}})
                print(json.dumps(out[-1]), flush=True)
                E.free()
        setenv(UPIR_JACOBI_ORDER=None, UPIR_JACOBI_CHUNK=None, UPIR_JACOBI_TEAMS=None, UPIR_JACOBI_POLICY=None)
    E.U.upir_finalize(E.ctx)


if __name__ == "__main__":
    main()
