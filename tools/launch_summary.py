"""Summarise an ncu launch list (gpu__time_duration.sum per launch) of
`bench.py` into profiles/<tag>_launch_summary.txt.

    python tools/launch_summary.py <tag> gpurun_out/launches.csv [bench line of an UNINSTRUMENTED run]
"""
import csv
import json
import os
import re
import sys
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    name = re.sub(r"\(.*", "", name)
    name = name[5:] if name.startswith("void ") else name
    return name.replace("upir::", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")


def main():
    tag, path = sys.argv[1], sys.argv[2]
    bench = None
    if len(sys.argv) > 3 and os.path.exists(sys.argv[3]):
        lines = [l for l in open(sys.argv[3]) if l.startswith("{")]
        bench = json.loads(lines[-1]) if lines else None
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr = rows[0]
    ik, iv, iu, ig = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit"), hdr.index("Grid Size")
    seq = []
    for r in rows[1:]:
        v = float(r[iv].replace(",", ""))
        v = v / 1e3 if r[iu] == "ns" else (v * 1e3 if r[iu] == "ms" else v)   # -> us
        seq.append((short(r[ik]), r[ig], v))
    groups = OrderedDict()
    for k, g, v in seq:
        groups.setdefault((k, g), []).append(v)
    out = [f"# Launch list of `python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline` under",
           "# (C5a reuses the C2 int64 kernel over 2^34 elements: its launches fall in the same row)",
           "# `ncu --metrics gpu__time_duration.sum --clock-control none` (cold-cache, serialised launches).",
           f"# Raw CSV: profiles/{tag}_launches.csv.  {len(seq)} launches.", "#",
           "# kernel (grid)                                              launches   avg us    total ms"]
    for (k, g), vs in groups.items():
        out.append(f"  {k[:58]:58s} {g:>14s} {len(vs):5d} {sum(vs) / len(vs):9.1f} {sum(vs) / 1e3:10.2f}")
    # C2 step: the reduce launches of the headline loop come first (warm-up +
    # timed steps, int64 / fp32 alternating); the C5a line later launches the
    # same int64 kernel over 2^34 elements, so only the leading run counts
    red = []
    for k, g, v in seq:
        if k.startswith("stream_loop_kernel<0, 2") or k.startswith("stream_loop_kernel<1, 2"):
            red.append((k, v))
        elif red and not k.startswith("synth_fill"):
            break
    i64 = [v for k, v in red if k.startswith("stream_loop_kernel<0")]
    f32 = [v for k, v in red if k.startswith("stream_loop_kernel<1")]
    if i64 and f32:
        a, b = sum(i64) / len(i64), sum(f32) / len(f32)
        out += ["#", "# C2 step (the bench line's `value`): two loop kernels per step",
                f"#   REDUCE int64 sum+max  avg {a:8.1f} us  ({100 * a / (a + b):.1f}% of the step)",
                f"#   REDUCE fp32  sum+max  avg {b:8.1f} us  ({100 * b / (a + b):.1f}% of the step)"]
        if bench and "kernel_ms" in bench:
            ka, kb = bench["kernel_ms"]["reduce_i64"], bench["kernel_ms"]["reduce_f32"]
            out.append(f"# bench.py CUDA events (warm, back to back): {ka:.3f} / {kb:.3f} ms -> "
                       f"{100 * ka / (ka + kb):.1f}% / {100 * kb / (ka + kb):.1f}% of the step")
    dst = os.path.join(ROOT, "profiles", f"{tag}_launch_summary.txt")
    open(dst, "w").write("\n".join(out) + "\n")
    print("wrote", dst)


if __name__ == "__main__":
    main()
