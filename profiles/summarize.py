"""Summarise ncu captures of K1 into profiles/ (run here, on CPU, after gpurun).

    python profiles/summarize.py <round-tag> <dir with k1_logp/k1_logp+H/k1_loss .ncu-rep> [launches.csv]

Writes profiles/<tag>_k1_ncu.md and profiles/k1_traffic.json (the per-launch DRAM
traffic bench.py reports as roofline.traffic).
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak (ncu)"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [{h: (r[i], units[i]) for i, h in enumerate(hdr)} for r in rows[2:]]


def main():
    tag, d = sys.argv[1], sys.argv[2]
    lines = [f"# K1 ncu summary ({tag})", "",
             "`ncu --set full --clock-control none --import-source on` on one launch of each K1 variant",
             "(tools/k1_bench.py: 8 sequences x 1024 tokens x V=128256 bf16 = 2.10 GB of logits per launch,",
             "the bench's launch shape; profiles/run_ncu_k1.sh).", ""]
    traffic = {}
    fwd = ("logp", "logp+H", "loss")
    for kind in fwd + ("lossgrad", "grad"):
        rep = os.path.join(d, f"k5_{kind}.ncu-rep" if kind == "grad" else f"k1_{kind}.ncu-rep")
        if not os.path.exists(rep):
            continue
        r = raw(rep)[0]
        name = r["Kernel Name"][0]
        lines += [f"## {kind}: `{name[:90]}`", "", "| metric | value |", "|---|---|"]
        for m, label in METRICS:
            if m in r:
                v, u = r[m]
                lines.append(f"| {label} (`{m}`) | {v} {u} |")
        rd = float(r["dram__bytes_read.sum"][0]) * (1e9 if r["dram__bytes_read.sum"][1] == "Gbyte" else 1e6 if r["dram__bytes_read.sum"][1] == "Mbyte" else 1)
        wr = float(r["dram__bytes_write.sum"][0]) * (1e9 if r["dram__bytes_write.sum"][1] == "Gbyte" else 1e6 if r["dram__bytes_write.sum"][1] == "Mbyte" else 1e3 if r["dram__bytes_write.sum"][1] == "Kbyte" else 1)
        t = float(r["gpu__time_duration.sum"][0]) * (1e-6 if r["gpu__time_duration.sum"][1] == "us" else 1e-9 if r["gpu__time_duration.sum"][1] == "ns" else 1e-3)
        alg = 8 * 1024 * 128256 * 2 * (1 if kind in fwd else 2)  # backward: + bf16 dlogits written
        lines += [f"| algorithmic logits bytes | {alg} |", f"| traffic / algorithmic | {(rd + wr) / alg:.4f} |",
                  f"| achieved (traffic / duration, under ncu) | {(rd + wr) / t / 1e9:.1f} GB/s |", ""]
        stalls = sorted(((float(v[0] or 0), k) for k, v in r.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_")
                         and not k.endswith("not_issued")), reverse=True)[:6]
        lines += ["top stall reasons (pc samples): " + ", ".join(f"{k.split('stalled_')[1]} {int(v)}" for v, k in stalls), ""]
        traffic[kind] = rd + wr
    if traffic:
        path = os.path.join(os.path.dirname(__file__), "k1_traffic.json")
        entry = {"V": 128256, "T": 1024, "mb": 8, "tag": tag,
                 "dram_bytes_per_launch": round(sum(traffic[k] for k in fwd if k in traffic) /
                                                max(1, sum(k in traffic for k in fwd))),
                 "per_variant": {k: round(v) for k, v in traffic.items()}}
        old = json.load(open(path)) if os.path.exists(path) else {}
        # keep the other launch shapes' captures (bench.py matches on V, T, mb)
        others = [e for e in old.get("configs", []) if (e["V"], e["T"], e["mb"]) != (128256, 1024, 8)]
        json.dump(dict(entry, configs=[entry] + others), open(path, "w"), indent=1)
    if len(sys.argv) > 3:
        rows = list(csv.reader(open(sys.argv[3])))
        i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
        hdr = rows[i]
        tot, cnt = {}, {}
        for r in rows[i + 1:]:
            if len(r) < len(hdr) or r[hdr.index("Metric Name")] != "gpu__time_duration.sum":
                continue
            n = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")
            tot[n] = tot.get(n, 0.0) + float(r[hdr.index("Metric Value")].replace(",", ""))
            cnt[n] = cnt.get(n, 0) + 1
        T = sum(tot.values())
        lines += ["## launch list (bench.py --steps 2 --warmup 3 under `ncu --metrics gpu__time_duration.sum`)", "",
                  "| kernel | launches | total | avg | share |", "|---|---|---|---|---|"]
        for n in sorted(tot, key=lambda k: -tot[k]):
            lines.append(f"| `{n}` | {cnt[n]} | {tot[n] / 1e3:.1f} us | {tot[n] / cnt[n] / 1e3:.2f} us | {tot[n] / T:.4f} |")
    open(os.path.join(os.path.dirname(__file__), f"{tag}_k1_ncu.md"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
