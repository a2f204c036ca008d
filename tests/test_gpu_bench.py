"""bench.py's JSON contract on the GPU (small configs, so the whole file runs in ~1 min):
the keys the driver and DESIGN.md section 7 rely on, the e2e statistics check, the
reference arm, and the N > 1 path (two ranks sharing the one GPU, re-launched by
bench.py itself under torch.distributed.run)."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, env=None, timeout=600):
    e = dict(os.environ, **(env or {}))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, env=e,
                       capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _bench("--config", "tiny", "--steps", "3", "--warmup", "3", "--legs", "llama8b:secondary",
               "--leg-steps", "2", "--ref-seqs", "4")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "clocks",
              "gpu_launches", "legs"):
        assert k in d, k
    assert d["status"] == "ORL_OK" and d["n_gpus"] == 1 and d["steps"] == 3 and d["value"] > 0
    assert d["gpu_launches"] == 3 + 5      # tiny: one micro-batch per pass, K3, 4 whitening/statistics kernels
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 0 and r["achieved"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    c = d["cpu_baseline"]
    assert c["kind"] == "oracle" and c["cores"] >= 1 and c["value"] > 0 and "sequences" in c["sample"]
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["stats_bit_identical_to_device_step"]
    assert "workload" in d["config"] and "tiny" in d["config"]["workload"]
    leg = d["legs"]["llama8b:secondary"]
    assert leg["status"] == "ORL_OK" and leg["roofline"]["frac"] > 0 and "U{T/16..T}" in leg["workload"]


def test_bench_reference_arm():
    d = _bench("--impl", "reference", "--config", "tiny", "--steps", "2", "--warmup", "1")
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.skipif(torch.cuda.device_count() < 1, reason="needs a GPU")
def test_bench_two_ranks_on_one_gpu():
    """--gpus 2 without torchrun: bench.py re-launches itself; both ranks share cuda:0
    (ORL_BENCH_SHARED_GPU, gloo + peer-memory C1/C2); strong scaling over token-balanced
    shards of the ragged secondary lengths."""
    d = _bench("--gpus", "2", "--config", "rpp8", "--batch", "8", "--lengths", "secondary", "--steps", "3",
               "--warmup", "3", "--legs", "", "--no-cpu", "--no-e2e", env={"ORL_BENCH_SHARED_GPU": "1"})
    assert d["n_gpus"] == 2 and d["status"] == "ORL_OK" and d["scaling"] == "strong"
    assert [p["rank"] for p in d["per_rank"]] == [0, 1]
    sh = d["config"]["shards"]
    assert sh[0][0] == 0 and sh[0][1] == sh[1][0] and sh[1][1] == 8
    assert sum(p["tokens"] for p in d["per_rank"]) == d["config"]["tokens_per_step"]
    assert "test_mode" in d
