"""Host-side logic of the N > 1 path (CPU, -m "not gpu"): the token-balanced,
group-aligned contiguous rank shards bench.py and a trainer use (SPEC S:468
"contiguous shards weighted by token counts")."""
import numpy as np
import pytest

from paper_2405_11143_b200 import synth


@pytest.mark.parametrize("name", ["llama8b", "longcot", "grpo", "rpp8"])
@pytest.mark.parametrize("n", [1, 2, 4, 8])
def test_token_balanced_shards(name, n):
    c = synth.CONFIGS[name]
    G = max(1, c["group_size"])
    for mode in ("full", synth.SECONDARY_LENGTHS[name]):
        L = synth.lengths_for(c["B"], c["T"], 1234, mode).numpy().astype(np.int64)
        b = synth.split_bounds_tokens(L, n, G)
        assert len(b) == n and b[0][0] == 0 and b[-1][1] == c["B"]
        assert all(b[r][1] == b[r + 1][0] for r in range(n - 1))          # contiguous, in order
        assert all((e - s) % G == 0 and e > s for s, e in b)               # whole groups, never empty
        tok = np.array([L[s:e].sum() for s, e in b], dtype=np.float64)
        gmax = L.reshape(-1, G).sum(axis=1).max()
        # the midpoint rule puts every cut within one group of the ideal token boundary
        assert tok.max() - tok.mean() <= gmax + 1e-9, (mode, tok)
        if mode == "full":
            assert np.all(tok == tok[0]) or c["B"] // G % n


def test_token_balanced_shards_edge_cases():
    # a huge first group: the others still get one group each
    L = np.array([1000, 1000, 1, 1, 1, 1, 1, 1])
    b = synth.split_bounds_tokens(L, 3, 2)
    assert b == [(0, 2), (2, 4), (4, 8)]
    # all-empty batch falls back to an even split of sequences
    assert synth.split_bounds_tokens(np.zeros(8), 4, 1) == synth.split_bounds(8, 4, 1)
    with pytest.raises(ValueError):
        synth.split_bounds_tokens(np.ones(7), 2, 2)


def _bench_cpu(args, env=None):
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    e = dict(os.environ, **(env or {}))
    return subprocess.run([sys.executable, os.path.join(root, "bench.py"), *args], cwd=root, env=e,
                          capture_output=True, text=True, timeout=600)


def test_bench_rejects_world_size_mismatch():
    """Under torchrun WORLD_SIZE must equal --gpus (a plain --gpus 8 never silently measures 1 GPU)."""
    r = _bench_cpu(["--gpus", "1"], env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE=2 but --gpus 1" in (r.stderr + r.stdout)


def test_bench_reference_arm_on_cpu():
    """--impl reference: the fp64 oracle on the host cores, one JSON line with the contract's keys."""
    import json
    r = _bench_cpu(["--impl", "reference", "--config", "tiny", "--steps", "2", "--warmup", "1"])
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "tokens/s" and d["dtype"] == "f64"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_clock_sampler_keeps_only_the_timed_region(tmp_path, monkeypatch):
    """bench.py's nvidia-smi sampler (CPU, with a stand-in nvidia-smi that starts slowly and
    then prints one sample every 50 ms): start() returns once sampling runs, and only
    samples between begin() and end() are reported -- a short timed region still gets some."""
    import os
    import sys
    import time

    fake = tmp_path / "nvidia-smi"
    fake.write_text("#!/bin/bash\nsleep 0.5\ni=0\nwhile true; do i=$((i+1));\n"
                    "  if [ -f " + str(tmp_path / "hot") + " ]; then c=1500; r=Active; else c=1965; r='Not Active'; fi\n"
                    "  echo \"$(date +'%Y/%m/%d %H:%M:%S.%3N'), 0, $c, 1965, 900.0, 0x0, Not Active, Not Active, "
                    "Not Active, $r\"; sleep 0.05; done\n")
    fake.chmod(0o755)
    monkeypatch.setenv("PATH", f"{tmp_path}{os.pathsep}{os.environ['PATH']}")
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import bench

    c = bench.ClockSampler(0).start()
    assert c.lines, "start() must wait for the first sample"
    time.sleep(0.3)                                  # samples before the timed region: 1965 MHz
    (tmp_path / "hot").write_text("")
    time.sleep(0.12)
    c.begin()
    time.sleep(0.25)                                 # the timed region: 1500 MHz, sw_power_cap
    c.end()
    (tmp_path / "hot").unlink()
    time.sleep(0.3)
    r = c.stop()
    assert r is not None and r["samples"] >= 3
    assert r["sm_mhz"] == 1500.0 and r["reasons"] == ["sw_power_cap"] and r["sm_max_mhz"] == 1965.0
    # a region shorter than the sampling interval reports the next sample
    c = bench.ClockSampler(0).start()
    c.begin()
    c.end()
    r = c.stop()                                     # waits for the sample after begin()
    assert r is not None and r["samples"] == 1
