"""Host-side logic of bench.py (no GPU): the launcher refuses to run fewer
ranks than --gpus asks for, the JSON line is strict JSON, and the summary
collects one entry per body / exchange path."""
import json
import math
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def _run(args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.pop("UPIR_BENCH_SHARED_GPU", None)
    e.update(env or {})
    e["CUDA_VISIBLE_DEVICES"] = ""   # this host has no GPU; make that explicit
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          env=e, timeout=300)


def test_gpus_n_refuses_without_n_gpus():
    r = _run(["--gpus", "2"])
    assert r.returncode == 2
    assert "refusing" in r.stderr and r.stdout == ""


def test_world_size_must_match_gpus():
    r = _run(["--gpus", "1"], {"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode == 2
    assert "WORLD_SIZE=2" in r.stderr


def test_clean_makes_strict_json():
    out = bench.clean({"a": float("nan"), "b": [1.0, float("inf")], "c": {"d": 2.5}})
    assert out == {"a": None, "b": [1.0, None], "c": {"d": 2.5}}
    json.loads(json.dumps(out, allow_nan=False))


def test_summary_one_entry_per_path_and_body():
    lines = {"c5a": {"paths": {"nccl": {"value": 1.0, "unit": "GB/s", "ms": 2.0, "frac": 0.5, "frac_8TB": 0.4,
                                        "rank_GB/s": 9.0},
                               "peer": {"unavailable": "x"}}},
             "c5b": {"error": "boom"}}
    kernels = {"axpy": {"summary": {"static": {"GB/s": 1.0}}}, "matmul": {"error": "e"}}
    s = bench.summarize(lines, kernels)
    assert s["c5a:nccl"] == {"value": 1.0, "unit": "GB/s", "ms": 2.0, "frac": 0.5, "frac_8TB": 0.4}
    assert s["c5a:peer"] == {"unavailable": "x"}
    assert s["c5b"] == {"error": "boom"}
    assert s["axpy:static"] == {"GB/s": 1.0}
    assert s["matmul"] == {"error": "e"}


def test_fracs_against_both_denominators():
    f = bench.fracs(4000.0, 6570.3)
    assert math.isclose(f["frac"], 4000.0 / 6570.3, rel_tol=1e-3)
    assert math.isclose(f["frac_8TB"], 0.5, rel_tol=1e-9)
