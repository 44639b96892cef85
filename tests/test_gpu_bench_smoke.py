"""bench.py end to end on the GPU at reduced sizes: every line of the JSON
runs (no "error" entries), the JSON is strict, and the multi-rank code runs
with --gpus 2 on one GPU (ranks sharing cuda:0; the NCCL lines report
"unavailable" there)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SMALL = {"UPIR_C5A_LOG2": "24", "UPIR_C5B_N": "2048"}


def _bench(args, env=None, timeout=900):
    e = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        e.pop(k, None)
    e.update(SMALL)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       env=e, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0], parse_constant=lambda c: pytest.fail(f"non-strict JSON constant {c}"))


def test_bench_n1_every_line_runs(upir):
    d = _bench(["--steps", "2", "--warmup", "1", "--e2e-steps", "1", "--n-log2", "24", "--no-cpu-baseline"])
    for k in ("metric", "value", "unit", "n_gpus", "ms_per_step", "roofline", "clocks", "e2e", "gpu_launches",
              "summary", "config"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] == 4
    bad = {k: v for k, v in d["summary"].items() if "error" in v}
    assert not bad, bad
    for key in ("C2:reduce_i64", "c5a:local", "c5b:local", "c5b:split_async", "axpy:static", "jacobi:C3",
                "matvec:matvec_16384", "stencil7:stencil7_8192", "matmul:C4_bf16", "matmul:C4_fp32"):
        assert key in d["summary"], key
    assert d["scaling_lines"]["c5a"]["results_identical_across_paths"]
    assert d["scaling_lines"]["c5b"]["rows_identical_across_paths"]
    assert d["e2e_pipelined"]["int64_results_equal_serial"]


def test_bench_reference_arm(upir):
    d = _bench(["--impl", "reference", "--steps", "1", "--warmup", "0"], env={"UPIR_REF_LOG2": "20"})
    assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "oracle" and d["ms_per_step"] > 0


def test_bench_two_ranks_on_one_gpu(upir):
    d = _bench(["--gpus", "2", "--steps", "2", "--warmup", "1", "--e2e-steps", "1", "--n-log2", "22",
                "--no-kernels"], env={"UPIR_BENCH_SHARED_GPU": "1"})
    assert d["n_gpus"] == 2
    s = d["summary"]
    assert "unavailable" in s["c5a:nccl"] and "unavailable" in s["c5b:nccl"]
    assert s["c5a:peer"]["value"] > 0 and s["c5b:peer"]["value"] > 0
    assert d["scaling_lines"]["c5b"]["rows_identical_across_paths"]
