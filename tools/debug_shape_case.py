"""Debug one case of tests/test_gpu_shapes.py: print the GPU advantages next to the oracle's
(stage-isolated) for the valid tokens.   python tools/debug_shape_case.py 170 222 ..."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2405_11143_b200 import orl, synth  # noqa: E402
from paper_2405_11143_b200.pipeline import Buffers, PathConfig, run_iteration  # noqa: E402
from tests import test_gpu_shapes as T  # noqa: E402
from tests.test_gpu_parity import _isolated_oracle, _np  # noqa: E402
from tests import parity  # noqa: E402

np.set_printoptions(precision=9, linewidth=200)
DEV = torch.device("cuda:0")
for i in map(int, sys.argv[1:]):
    cs = T._case(i)
    V, B, Tn, kind, G = cs["V"], cs["B"], cs["T"], cs["kind"], cs["G"]
    c = dict(synth.CONFIGS["tiny"], V=V, T=Tn, adv_kind=kind, group_size=G)
    if kind == "grpo":
        c.update(kl_mode="loss", kl_est_loss="k2", beta_loss=0.05, whiten=False, eps_v=0.0, c1=0.0)
    if kind.startswith("rpp"):
        c.update(eps_v=0.0, c1=0.0)
    batch = synth.make_batch(i, B, Tn, V, cs["dtype"], "stress", cs["L"], "group_bernoulli" if G > 1 else "normal", G)
    cfg = PathConfig.from_synth(c)
    cfg.inv_temp = cs["inv_temp"]
    g = {k: (v.to(DEV) if isinstance(v, torch.Tensor) else v) for k, v in batch.items()}
    src = lambda role, s, e: g[f"logits_{role}"][s:e]  # noqa: E731
    ctx = orl.Context(0)
    bufs = Buffers(B, Tn, DEV, G)
    status, st = run_iteration(ctx, g, cfg, bufs, src, mb=cs["mb"])
    torch.cuda.synchronize()
    npb = synth.batch_to_numpy(batch)
    m = parity.valid_mask(npb["lengths"], Tn)
    ocfg = dict(c, kl_mode=c.get("kl_mode", "reward"))
    ocfg["inv_temp"] = cs["inv_temp"]
    out_i, glob_i = _isolated_oracle(npb, bufs, ocfg)
    print(f"case {i}: kind {kind} B {B} T {Tn} L {list(npb['lengths'])} R {npb['seq_reward']} gamma {c['gamma']} lam {c['lam']}")
    print("  shaped gpu   ", _np(bufs.shaped)[m])
    print("  adv gpu      ", _np(bufs.adv)[m])
    print("  adv oracle   ", out_i[0]["adv"][m])
    if out_i[0].get("ret") is not None:
        print("  ret gpu      ", _np(bufs.ret)[m])
        print("  ret oracle   ", out_i[0]["ret"][m])
    if "values_old" in npb:
        print("  values_old   ", npb["values_old"][m])
    ctx.close()
