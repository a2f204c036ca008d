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
    for n in VARIANTS:
        so = os.path.join(OUT, f"liborl_{n}.so")
        if not os.path.exists(so):
            continue
        env = dict(os.environ, ORL_LIB_PATH=so)
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "k1_bench.py"), "--kinds", "logp,logp+H,loss"],
                             env=env, capture_output=True, text=True)
        print(f"== {n}\n{out.stdout}{out.stderr[-500:] if out.returncode else ''}", flush=True)
