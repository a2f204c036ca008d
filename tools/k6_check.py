"""Quick NEXT-4 diagnostics on one small case: GEMM (gathered z_y) vs a torch fp32
matmul, and logp/H/lse vs the same torch reference (not the oracle; for debugging).
    python tools/k6_check.py [B T d V]"""
import sys

import torch

from paper_2405_11143_b200 import orl, synth

B, T, d, V = (int(x) for x in sys.argv[1:5]) if len(sys.argv) > 4 else (2, 64, 128, 512)
dev = torch.device("cuda:0")
b = synth.make_lmhead_batch(3, B, T, d, V, lengths="full", device=dev)
ctx = orl.Context(0)
tok, L = b["tokens"].to(dev), b["lengths"].to(dev)
out = {k: torch.zeros(B, T, device=dev) for k in ("logp", "entropy", "lse", "gathered")}
orl.orl_begin_iteration(ctx)
orl.orl_lmhead_logprobs(ctx, tok, L, b["hidden_old"], b["weight"], out["logp"], entropy=out["entropy"],
                        lse=out["lse"], gathered=out["gathered"])
torch.cuda.synchronize()
z = b["hidden_old"].float() @ b["weight"].float().T          # [B*T, V]
y = tok.reshape(-1).long()
zy = z.gather(1, y[:, None])[:, 0]
ls = torch.log_softmax(z.double(), 1)
ref = {"gathered": zy, "lse": torch.logsumexp(z.double(), 1), "logp": ls.gather(1, y[:, None])[:, 0],
       "entropy": -(ls.exp() * ls).sum(1)}
for k, r in ref.items():
    g = out[k].reshape(-1).double()
    err = (g - r.double()).abs()
    print(f"{k:9s} max err {err.max().item():.3e}  at row {int(err.argmax())}  gpu {g[int(err.argmax())].item():.6f} ref {r[int(err.argmax())].item():.6f}")
# which vocab column does the GPU's gathered value match?
r0 = 0
m = (z[r0] - out["gathered"].reshape(-1)[r0]).abs().argmin()
print("row 0: y =", int(y[r0]), "gathered matches column", int(m))
print(orl.orl_finalize(ctx, orl.PPOConfig()))
