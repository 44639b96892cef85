"""Sweep: C3 Jacobi (8192^2, 100 sweeps, one graph) over teams x tile x ring
depth (UPIR_JACOBI_NST; 0 = the launcher's choice).  Run on the GPU box:
python tools/experiments/jacobi_sweep.py"""
import os
import sys
import types

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2209_10643_b200 as U  # noqa: E402


def main():
    ctx = U.upir_init(0)
    stream = torch.cuda.ExternalStream(U.upir_ctx_stream(ctx, 0))
    peaks, src = bench.measured_peaks()
    args = types.SimpleNamespace(steps=5)
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
                    r = bench.bench_jacobi(args, U, ctx, stream, peaks, src)
                    print(f"tile {tile} teams {teams} nst {nst}: {r['GLUP/s']:.1f} GLUP/s "
                          f"frac {r['roofline']['frac']:.3f}", flush=True)
                except Exception as e:  # report, keep sweeping
                    print(f"tile {tile} teams {teams} nst {nst}: error {e}", flush=True)
    U.upir_finalize(ctx)


if __name__ == "__main__":
    main()
