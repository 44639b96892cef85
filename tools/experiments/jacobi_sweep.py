"""Sweep: C3 Jacobi (8192^2, 100 sweeps, one graph) over teams x tile x ring
depth (UPIR_JACOBI_NST; 0 = the launcher's choice).  Run on the GPU box:
python tools/experiments/jacobi_sweep.py"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def main():
    E = bench.Env(argparse.Namespace(gpus=1, steps=5, warmup=3, impl="upir", sched="static", n_log2=30,
                                     e2e_steps=0, no_cpu_baseline=True, no_kernels=False, no_scaling=True, lines=None))
    tiles = os.environ.get("TILES", "16x256,32x256").split(",")
    teams_l = [int(t) for t in os.environ.get("TEAMS", "148,296,444").split(",")]
    nsts = os.environ.get("NSTS", "0,2,3,4").split(",")
    for tile in tiles:
        for teams in teams_l:
            for nst in nsts:
                os.environ["UPIR_JACOBI_TILE"] = tile
                os.environ["UPIR_JACOBI_TEAMS"] = str(teams)
                os.environ["UPIR_JACOBI_NST"] = nst
                try:
                    r = bench.bench_jacobi(E)
                    print(f"tile {tile} teams {teams} nst {nst}: {r['GLUP/s']:.1f} GLUP/s "
                          f"frac {r['roofline']['frac']:.3f}", flush=True)
                except Exception as e:  # report, keep sweeping
                    print(f"tile {tile} teams {teams} nst {nst}: error {e}", flush=True)
                E.free()
    E.U.upir_finalize(E.ctx)


if __name__ == "__main__":
    main()
