"""Build K1 launch-shape variants (here) and benchmark them (on the GPU box).

    python tools/k1_tune.py build      # nvcc variants into build/tune/
    python tools/k1_tune.py run        # k1_bench.py for each variant
"""
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
VARIANTS = {
    "default": [],
    "always_ent": ["ORL_K1_ALWAYS_ENT=1"],
    # K6 (NEXT-4) wait policies: epilogue / producer mbarrier suspend hints (ns)
    "k6_spin": ["ORL_K6_EPI_SLEEP_NS=0", "ORL_K6_PROD_SLEEP_NS=0"],
    "k6_epi2k": ["ORL_K6_EPI_SLEEP_NS=2000"],
    "k6_epi20k": ["ORL_K6_EPI_SLEEP_NS=20000"],
    "k6_epi20k_prod1k": ["ORL_K6_EPI_SLEEP_NS=20000", "ORL_K6_PROD_SLEEP_NS=1000"],
    "k6_nomath": ["ORL_K6_EPI_NOMATH=1"],
    # K1 launch shapes for the power-capped (sustained) regime
    "cw8": ["ORL_K1_CONSUMER_WARPS=8"],
    "cw8_c16k": ["ORL_K1_CONSUMER_WARPS=8", "ORL_K1_CHUNK=16384", "ORL_K1_STAGES=12"],
    "cw8_mb2": ["ORL_K1_CONSUMER_WARPS=8", "ORL_K1_MINBLOCKS=2", "ORL_K1_STAGES=3"],
    "s4": ["ORL_K1_STAGES=4"],
    "s5": ["ORL_K1_STAGES=5"],
    "epi3_s5": ["ORL_K1_EPI_WARPS=3", "ORL_K1_STAGES=5"],
    "epi4_s5": ["ORL_K1_EPI_WARPS=4", "ORL_K1_STAGES=5"],
    # suspend-time hints on the epilogue's row wait / the consumers' stage wait (ns)
    "ew20k": ["ORL_K1_EPI_WAIT_NS=20000"],
    "ew2k": ["ORL_K1_EPI_WAIT_NS=2000"],
    "cw1k": ["ORL_K1_CONS_WAIT_NS=1000"],
    "ew20k_cw1k": ["ORL_K1_EPI_WAIT_NS=20000", "ORL_K1_CONS_WAIT_NS=1000"],
}
OUT = os.path.join(ROOT, "build", "tune")

if sys.argv[1] == "build":
    from paper_2405_11143_b200 import build
    os.makedirs(OUT, exist_ok=True)
    names = sys.argv[2:] or list(VARIANTS)
    with ThreadPoolExecutor(len(names)) as ex:
        list(ex.map(lambda n: build.build(force=True, defines=VARIANTS[n], out=os.path.join(OUT, f"liborl_{n}.so")), names))
    print("built", names)
else:
    for n in (sys.argv[2:] or VARIANTS):
        so = os.path.join(OUT, f"liborl_{n}.so")
        if not os.path.exists(so):
            continue
        env = dict(os.environ, ORL_LIB_PATH=so)
        cmd = [sys.executable, os.path.join(ROOT, "tools", "k1_bench.py"), "--kinds", "logp,logp+H,loss"]
        if n.startswith("k6"):
            cmd = [sys.executable, os.path.join(ROOT, "tools", "k6_bench.py"), "--reps", "300", "--no-baseline"]
        out = subprocess.run(cmd, env=env, capture_output=True, text=True)
        print(f"== {n}\n{out.stdout}{out.stderr[-500:] if out.returncode else ''}", flush=True)
