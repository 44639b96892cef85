"""Summarise ncu reports into profiles/ (run here, on the CPU box).

    python tools/ncu_summary.py <round-tag> gpurun_out/prof_*.ncu-rep
    (env UPIR_PROFILES_OUT=<dir> writes there instead of profiles/)

Writes profiles/<tag>_<name>.txt (key metrics per profiled kernel launch)
and updates profiles/traffic.json (DRAM bytes per launch, read by bench.py).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.environ.get("UPIR_PROFILES_OUT", os.path.join(ROOT, "profiles"))
KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__cycles_elapsed.avg.per_second",
    "l1tex__t_bytes.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {h: (v, u) for h, v, u in zip(hdr, r, units)}
        res.append(d)
    return res


def fnum(v):
    try:
        return float(v.replace(",", ""))
    except Exception:
        return None


def to_bytes(v, u):
    x = fnum(v)
    if x is None:
        return None
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    return x * scale.get(u, 1)


def main():
    tag = sys.argv[1]
    os.makedirs(OUT, exist_ok=True)
    traffic_path = os.path.join(OUT, "traffic.json")
    if not os.path.exists(traffic_path) and os.path.exists(os.path.join(ROOT, "profiles", "traffic.json")):
        traffic_path_in = os.path.join(ROOT, "profiles", "traffic.json")
    else:
        traffic_path_in = traffic_path
    traffic = json.load(open(traffic_path_in)) if os.path.exists(traffic_path_in) else {}
    for rep in sys.argv[2:]:
        name = os.path.basename(rep).replace(".ncu-rep", "").replace("prof_", "")
        launches = raw(rep)
        lines = [f"# ncu --set full summary: {os.path.basename(rep)} (round tag {tag})",
                 "# command: see tools/prof_all.sh; --clock-control none; per-launch values"]
        for i, d in enumerate(launches):
            kname = d.get("Kernel Name", ("?", ""))[0]
            lines.append(f"\n## launch {i}: {kname[:160]}")
            for k in KEYS:
                if k in d:
                    lines.append(f"{k} = {d[k][0]} {d[k][1]}")
            rb = to_bytes(*d["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in d else None
            wb = to_bytes(*d["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in d else None
            if rb is not None and wb is not None:
                lines.append(f"dram_traffic_bytes = {rb + wb:.0f}")
                key = name   # the profile name of tools/prof_all.sh (= the bench's traffic key)
                if key and key not in traffic.get("_seen_" + tag, []):
                    traffic[key] = rb + wb
                    traffic.setdefault("_seen_" + tag, []).append(key)
        out = os.path.join(OUT, f"{tag}_{name}.txt")
        with open(out, "w") as f:
            f.write("\n".join(lines) + "\n")
        print("wrote", out)
    traffic = {k: v for k, v in traffic.items() if not k.startswith("_seen_")}
    traffic["_note"] = ("dram__bytes_read.sum + dram__bytes_write.sum per launch from ncu --set full "
                        f"(tag {tag}); see profiles/{tag}_*.txt")
    json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)
    print("wrote", traffic_path)


if __name__ == "__main__":
    main()
