#!/usr/bin/env python
"""Benchmark of the logits -> PPO-loss path (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config grpo] [--impl ours|reference]
                    [--scaling strong|weak] [--lengths full|secondary] [--legs ...]

One step = one PPO/GRPO iteration of the whole hot path on every rank (S1 old,
S1+S2+S3 ref, S4/S5 advantages, S6 + collective C1, S1+S7..S9 actor, S10 +
collective C2) over a synthetic rollout of the named BASELINE.json
configuration.  Default: configs[3], "grpo" (256 prompts x 8 samples, T=4096,
V=128256 bf16, GRPO group advantages, k2 KL in the loss) -- the largest
single-GPU configuration of BASELINE.json.  Its 3 x 2.15 TB of logits do not
fit in HBM, so every micro-batch streams from a pool of micro-batch buffers per
model (8.4 GB each, >> the 126 MB L2: every read is an HBM read).

N > 1: one process per GPU.  `--gpus N` without WORLD_SIZE re-launches itself
under torch.distributed.run (127.0.0.1); under torchrun WORLD_SIZE must equal
--gpus.  --scaling strong (default): the config's global batch is split into N
contiguous, group-aligned shards balanced by valid tokens;
--scaling weak: every rank holds the config's whole batch.

Prints ONE JSON line on rank 0 (see DESIGN.md section 7 for every field).  The
headline config is followed by short legs on the other shapes (`legs`): the
Llama-3 config with the NEXT-1 / NEXT-4 / CUDA-graph measurements, long-CoT,
the north star's V=128256/T=8192 target shape, and ragged (secondary) lengths.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

METRIC = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
UNIT = "tokens/s"
SIDE_BYTES = {"old": 8, "ref": 8 + 12, "new": 8 + 28 + 16 + 1}   # side bytes per token and pass (DESIGN 5.1)
LEGS_DEFAULT = "llama8b,longcot,target,llama8b:secondary,longcot:secondary"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    except (OSError, ValueError, KeyError, TypeError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def _bf16_peak(sustained: bool):
    """Dense bf16 tensor peak in TFLOP/s: MEASURED_PEAKS.json (cuBLAS, burst or the
    seconds-long power-capped loop), else the profiling guide's fallback."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    key = "bf16_tflops_sustained" if sustained else "bf16_tflops"
    try:
        return float(json.load(open(p))[key]), f"measured (MEASURED_PEAKS.json {key}, cuBLAS)"
    except (OSError, ValueError, KeyError, TypeError):
        pass
    return (1400.0, "fallback sustained (B200_PROFILING.md ~1.4 PFLOP/s under the power cap)") if sustained else \
        (1590.0, "fallback burst (B200_PROFILING.md 1.59 PFLOP/s)")


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _lengths_mode(name, lengths):
    from paper_2405_11143_b200 import synth
    return "full" if lengths == "full" else synth.SECONDARY_LENGTHS.get(name, "mixed")


def _workload_desc(name, c, W):
    lm = {"full": "all L_b = T", "mixed": "L_b ~ U{T/16..T}", "cot": "40% L_b = T, rest U{T/8..T}"}[W["lengths"]]
    res = (f"pool of {W['pool']} micro-batch buffers per model (the batch's logits do not fit in HBM; "
           f"micro-batch k reads slot k mod {W['pool']})") if W["pool"] else "x3 models resident in HBM"
    return (f"{name}: B={W['B_rank']}/rank of {W['B_global']} T={c['T']} V={c['V']} {c['dtype']} logits {res}, "
            f"adv={c['adv_kind']} gamma={c['gamma']} lambda={c['lam']} whiten={c['whiten']} "
            f"eps=({c['eps_low']},{c['eps_high']}) eps_v={c['eps_v']} kl={c.get('kl_mode', 'reward')}, "
            f"micro-batch {c['mb']} seq, {lm}")


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi samples (every 50 ms) of SM clock, power and throttle reasons, kept for
    the timed region only, by nvidia-smi's own sample timestamps (a reader thread may see a
    line late).  start() returns once the first sample has arrived (nvidia-smi takes ~1 s to
    start); call it before the ranks' barrier so the wait does not skew the ranks' start.
    A region shorter than the sampling interval reports the first sample after its start."""
    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []
        self.t0 = self.t1 = None

    def start(self, wait_s: float = 10.0):
        import threading

        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return self
        first = threading.Event()

        def reader():
            for line in self.proc.stdout:
                self.lines.append((time.time(), line))
                first.set()

        self.thread = threading.Thread(target=reader, daemon=True)
        self.thread.start()
        first.wait(wait_s)
        return self

    def begin(self):
        self.t0 = time.time()

    def end(self):
        self.t1 = time.time()

    @staticmethod
    def _stamp(field, t_read):
        import datetime
        try:
            return datetime.datetime.strptime(field.strip(), "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except ValueError:
            return t_read

    def stop(self):
        if self.proc is None:
            return None
        # a region shorter than the sampling interval: let the first sample after its start arrive
        deadline = time.time() + 1.0
        t0 = self.t0 if self.t0 is not None else -1e300
        while time.time() < deadline and not (
                self.lines and self._stamp(self.lines[-1][1].split(",")[0], self.lines[-1][0]) >= t0):
            time.sleep(0.02)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.thread.join(timeout=5)
        rows = []
        for t_read, line in self.lines:
            f = [x.strip() for x in line.split(",")]
            if len(f) < 10:
                continue
            try:
                rows.append((self._stamp(f[0], t_read), float(f[2]), float(f[3]), float(f[4]), f[6:10]))
            except ValueError:
                continue
        t0 = self.t0 if self.t0 is not None else -1e300
        t1 = self.t1 if self.t1 is not None else 1e300
        inside = [r for r in rows if t0 <= r[0] <= t1]
        if not inside:                     # shorter than the sampling interval: the next sample
            after = [r for r in rows if t0 <= r[0] <= t1 + 0.5]
            inside = after[:1]
        if not inside:
            return None
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = {n for r in inside for n, v in zip(names, r[4]) if v.lower() == "active"}
        return {"sm_mhz": statistics.median(r[1] for r in inside), "sm_max_mhz": inside[-1][2],
                "reasons": sorted(reasons), "samples": len(inside),
                "power_w_median": statistics.median(r[3] for r in inside)}


# ----------------------------------------------------------------------------- oracle (CPU) leg
def _oracle_sample(logits_fn, batch_np, c, n_seq, cores):
    """Time the fp64 oracle on the first n_seq sequences: S1 for the three models
    (rows split over `cores` threads; ctypes releases the GIL), then the rest of
    the pipeline.  Returns (tokens, seconds)."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor

    sh = {k: v[:n_seq] for k, v in batch_np.items()}
    T = sh["tokens"].shape[1]
    t0 = time.perf_counter()
    for role in ("old", "ref", "new"):
        x = logits_fn(role, n_seq)                       # host [n_seq, T, V]
        flat = x.reshape(n_seq * T, 1, x.shape[-1])
        tok = sh["tokens"].reshape(-1, 1)
        ones = np.minimum(np.arange(T)[None, :] < sh["lengths"][:, None], 1).astype(np.int32).reshape(-1)
        parts = np.array_split(np.arange(n_seq * T), cores)

        def work(idx):
            if idx.size == 0:
                return idx, None
            return idx, oracle.logprobs(flat[idx[0]:idx[-1] + 1], tok[idx[0]:idx[-1] + 1], ones[idx[0]:idx[-1] + 1])

        lp = np.zeros(n_seq * T)
        ent = np.zeros(n_seq * T)
        with ThreadPoolExecutor(cores) as ex:
            for idx, o in ex.map(work, parts):
                if o is not None:
                    lp[idx] = o["logp"][:, 0]
                    ent[idx] = o["entropy"][:, 0]
        sh[f"logp_{role}"] = lp.reshape(n_seq, T)
        if role == "new":
            sh["entropy_new"] = ent.reshape(n_seq, T)
    oracle.pipeline([sh], c)
    dt = time.perf_counter() - t0
    return int(np.minimum(sh["lengths"], T).sum()), dt


def run_reference(args):
    """--impl reference: the fp64 oracle on the host cores, bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2405_11143_b200 import synth

    c = dict(synth.CONFIGS[args.config])
    T, V = c["T"], c["V"]
    G = max(1, c["group_size"])
    n_seq = max(G, (args.ref_seqs // G) * G)               # whole groups (GRPO)
    cap = min(T, -(-(args.ref_seqs * min(T, 1024)) // n_seq))  # ~ref_seqs x 1024 valid tokens per step
    cores = len(os.sched_getaffinity(0))
    dev = torch.device("cuda:0") if torch.cuda.is_available() else torch.device("cpu")
    # only the first `cap` positions of each response are in the sample: generate [n_seq, cap, V]
    batch = synth.make_batch(1234, n_seq, cap, V, c["dtype"], "realistic", "full", c["rewards"],
                             c["group_size"], device=dev)
    bnp = synth.batch_to_numpy(batch)
    fn = lambda role, n: bnp[f"logits_{role}"][:n]  # noqa: E731
    times, toks = [], 0
    for i in range(args.warmup + args.steps):
        toks, dt = _oracle_sample(fn, {k: v for k, v in bnp.items() if not k.startswith("logits_")}, c, n_seq, cores)
        if i >= args.warmup:
            times.append(dt)
    mean = sum(times) / len(times)
    val = toks / mean
    sample = (f"{n_seq} sequences ({n_seq // G} whole group(s)) of {args.config} with lengths capped at {cap} "
              f"({toks} tokens, 3 x {toks} vocab rows of V={V}), per step")
    line = {"impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean * 1e3, "higher_is_better": True,
            "scaling": args.scaling if args.gpus > 1 else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: T={T} V={V} {c['dtype']} logits, adv={c['adv_kind']} "
                                   "(oracle sample on the host cores)",
                       "global_batch": n_seq, "seq_len": T, "parallelism": "host threads"},
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": sample,
                             "cpu_model": _cpu_model()},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- workloads
def make_workload(name, args, env, lengths="full", scaling="strong", batch_override=0):
    """A synthetic rollout of config `name` for this rank: per-token inputs on the
    device and a logits source (resident buffers, or a pool of micro-batch buffers)."""
    from paper_2405_11143_b200 import synth
    from paper_2405_11143_b200.pipeline import Buffers, PathConfig

    world, rank, dev = env["world"], env["rank"], env["dev"]
    c = dict(synth.CONFIGS[name])
    T, V, mb, G = c["T"], c["V"], c["mb"], max(1, c["group_size"])
    lmode = _lengths_mode(name, lengths)
    tdt = torch.bfloat16 if c["dtype"] == "bf16" else torch.float32
    elt = 2 if tdt == torch.bfloat16 else 4
    seed = 1234
    if scaling == "weak":
        B_global = (batch_override or c["B"]) * world
        seed = 1234 + rank
        B_rank = batch_override or c["B"]
        L = synth.lengths_for(B_rank, T, seed, lmode)
        s0 = 0
        tok = synth.tokens_for(B_rank, T, V, seed)
        R = synth.rewards_for(B_rank, seed, c["rewards"], G)
        v_old, v_new = synth.values_for(B_rank, T, seed)
        bounds = None
    else:
        B_global = batch_override or c["B"]
        L_all = synth.lengths_for(B_global, T, seed, lmode)
        bounds = synth.split_bounds_tokens(L_all.numpy(), world, G)
        s0, e0 = bounds[rank]
        B_rank = e0 - s0
        L = L_all[s0:e0].clone()
        tok = synth.tokens_for(B_global, T, V, seed)[s0:e0].clone()
        R = synth.rewards_for(B_global, seed, c["rewards"], G)[s0:e0].clone()
        v_old, v_new = (v[s0:e0].clone() for v in synth.values_for(B_global, T, seed))
    n_mb = -(-B_rank // mb)
    full_bytes = 3 * B_rank * T * V * elt
    # ranks sharing one GPU (ORL_BENCH_SHARED_GPU functional test) split its memory
    free = torch.cuda.mem_get_info()[0] / (world if env["shared"] else 1)
    pooled = full_bytes > 0.80 * free
    pool = 0
    if pooled:
        # 2 buffers per model, 8.4 GB each at grpo (>> L2): micro-batch k reads slot k % 2;
        # token ids follow the slot, so each micro-batch's targets match its logits
        per_mb = mb * T * V * elt
        pool = max(1, min(n_mb, args.pool, int(0.70 * free // (3 * per_mb))))
        for k in range(pool, n_mb):
            a, b = k * mb, min(B_rank, (k + 1) * mb)
            j = (k % pool) * mb
            tok[a:b] = tok[j:j + (b - a)]
    tok, L, R, v_old, v_new = (x.to(env["dev"]) for x in (tok, L, R, v_old, v_new))
    if pooled:
        bufs_l = {r: torch.empty(pool * mb, T, V, dtype=tdt, device=dev) for r in synth.ROLES}
        for k in range(pool):
            sl = slice(k * mb, (k + 1) * mb)
            synth.fill_logits_(tuple(bufs_l[r][sl] for r in synth.ROLES), tok[sl], seed, rank * 100_000 + k,
                               "realistic")

        def src(role, s, e):
            k = (s // mb) % pool
            return bufs_l[role][k * mb:k * mb + (e - s)]
    else:
        bufs_l = {r: torch.empty(B_rank, T, V, dtype=tdt, device=dev) for r in synth.ROLES}
        for s in range(0, B_rank, mb):
            e = min(B_rank, s + mb)
            synth.fill_logits_(tuple(bufs_l[r][s:e] for r in synth.ROLES), tok[s:e], seed,
                               rank * 100_000 + s // mb, "realistic")
        src = lambda role, s, e: bufs_l[role][s:e]  # noqa: E731
    batch = dict(tokens=tok, lengths=L, seq_reward=R, values_old=v_old, values_new=v_new)
    return dict(name=name, c=c, cfg=PathConfig.from_synth(c), batch=batch, logits=bufs_l, src=src, pool=pool,
                B_rank=B_rank, B_global=B_global, T=T, V=V, mb=mb, elt=elt, n_mb=n_mb, lengths=lmode,
                bufs=Buffers(B_rank, T, dev, c["group_size"]), bounds=bounds, shard_start=s0,
                n_tok=int(L.clamp(0, T).sum().item()), step_bytes=3 * int(L.clamp(0, T).sum().item()) * V * elt)


def free_workload(W):
    for k in ("logits", "batch", "bufs", "src"):
        W.pop(k, None)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def timed_steps(ctx, W, env, steps, warmup, pdl_chain=True):
    """W untimed steps, then K steps between barrier + synchronize; CUDA events on the
    launching stream around every step and around each pass's back-to-back K1 launches."""
    from paper_2405_11143_b200.pipeline import run_iteration

    dist = env["dist"]
    stream = torch.cuda.current_stream()
    events, cur = [], {}

    def hook(tag):
        if cur.get("tag") != tag:
            a = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            cur.update(tag=tag, start=a, n=0)

        def done():
            cur["n"] += 1
            if cur["n"] == W["n_mb"]:
                b = torch.cuda.Event(enable_timing=True)
                b.record(stream)
                events.append((tag, cur["n"], cur["start"], b))
                cur.clear()
        return done

    def step(timing):
        return run_iteration(ctx, W["batch"], W["cfg"], W["bufs"], W["src"], W["mb"], stream=stream,
                             on_k1=hook if timing else None, pdl_chain=pdl_chain)

    status, st = None, None
    for _ in range(warmup):
        status, st = step(False)
    torch.cuda.synchronize()
    clocks = ClockSampler(env["local"]).start()   # before the barrier: its start-up wait is not timed
    if env["dist_mode"]:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.begin()
    l0 = ctx.launch_count
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    evs[0].record(stream)
    for i in range(steps):
        status, st = step(True)
        evs[i + 1].record(stream)
    torch.cuda.synchronize()
    clocks.end()
    if env["dist_mode"]:
        dist.barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(steps)]
    ms_rank = evs[0].elapsed_time(evs[-1]) / steps
    ms = ms_rank
    per_rank = None
    if env["dist_mode"]:
        tt = torch.tensor([ms_rank, float(W["n_tok"])], device=env["dev"], dtype=torch.float64)
        gathered = [torch.zeros_like(tt) for _ in range(env["world"])]
        dist.all_gather(gathered, tt)
        per_rank = [{"rank": r, "ms_per_step": round(float(g[0]), 4), "tokens": int(g[1]),
                     "tokens_per_s": round(float(g[1]) / (float(g[0]) / 1e3), 1)} for r, g in enumerate(gathered)]
        ms = max(float(g[0]) for g in gathered)
        total_tokens = int(sum(float(g[1]) for g in gathered))
    else:
        total_tokens = W["n_tok"]
    launches = (ctx.launch_count - l0) // steps
    return dict(ms=ms, ms_rank=ms_rank, per_step=per_step, events=events, launches=launches, status=status,
                stats=st, clocks=clk, total_tokens=total_tokens, per_rank=per_rank, steps=steps, warmup=warmup)


def roofline(W, R):
    """K1 (the dominant kernel) against the HBM peak: algorithmic bytes = valid tokens x
    (V x elt of logits + side arrays) per pass, over its event-timed duration."""
    steps = R["steps"]
    k1_ms = sum(a.elapsed_time(b) for _, _, a, b in R["events"])
    stage = {}
    for tag, _, a, b in R["events"]:
        stage[tag] = stage.get(tag, 0.0) + a.elapsed_time(b) / steps
    byts = sum(W["n_tok"] * (W["V"] * W["elt"] + SIDE_BYTES[tag]) for tag, _, _, _ in R["events"])
    n_k1 = sum(n for _, n, _, _ in R["events"])
    achieved = byts / (k1_ms / 1e3) / 1e9
    peak, peak_src = _peaks()
    traffic, traffic_src = None, None
    prof = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(prof):
        try:
            pj = json.load(open(prof))
            for e in pj.get("configs", [pj]):   # one ncu capture per (V, T, micro-batch, lengths) launch shape
                if e.get("V") == W["V"] and e.get("T") == W["T"] and e.get("mb") == W["mb"] and \
                        e.get("lengths", "full") == W["lengths"]:
                    traffic = e["dram_bytes_per_launch"]
                    traffic_src = e.get("tag")
        except Exception:
            traffic = None
    ms_rank = R["ms_rank"]
    stage_ms = {"S1_old": round(stage.get("old", 0.0), 4), "S1-S3_ref": round(stage.get("ref", 0.0), 4),
                "S1_S7-S9_actor": round(stage.get("new", 0.0), 4),
                "S4-S6_C1_S10_C2_and_gaps": round(ms_rank - sum(stage.values()), 4)}
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic, "traffic_capture": traffic_src,
            "kernel": "k1_tma_kernel (S1 + epilogues)", "launches_per_step": n_k1 // steps,
            "algorithmic_bytes_per_launch": int(byts / max(n_k1, 1)),
            "bytes_per_token": {t: W["V"] * W["elt"] + SIDE_BYTES[t] for t in ("old", "ref", "new")},
            "k1_share_of_step": round(k1_ms / (ms_rank * steps), 4), "peak_source": peak_src}, stage_ms


def _stats_round(st):
    return {k: (round(v, 6) if isinstance(v, float) else v) for k, v in st.items()}


# ----------------------------------------------------------------------------- our arm
def setup_env(args):
    import torch.distributed as dist

    from paper_2405_11143_b200 import orl

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}")
    # ORL_BENCH_SHARED_GPU=1 (functional test of the N > 1 code path on a one-GPU box; its
    # timings are not measurements): every rank on cuda:0, gloo process group, no NCCL
    # communicator (two ranks cannot share a GPU in NCCL), C1/C2 over the peer kernels.
    shared = os.environ.get("ORL_BENCH_SHARED_GPU") == "1" and world > 1
    if shared:
        local = 0
    elif local >= torch.cuda.device_count():
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local} but only {torch.cuda.device_count()} GPU(s)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    # under torchrun (even with one rank) use the distributed plumbing: NCCL process
    # group, unique-id broadcast, liborl NCCL communicator, barriers, max over ranks
    dist_mode = "WORLD_SIZE" in os.environ
    if shared:
        dist.init_process_group("gloo")
        ctx = orl.Context(local, world, rank, None)
    elif dist_mode:
        dist.init_process_group("nccl", device_id=dev)
        uid = [orl.orl_get_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        ctx = orl.Context(local, world, rank, uid[0])
    else:
        ctx = orl.Context(local)
    return dict(world=world, rank=rank, local=local, dev=dev, dist=dist, dist_mode=dist_mode, shared=shared, ctx=ctx)


def choose_collective(args, env, W):
    """C1/C2 transport at N > 1: the single-kernel peer-memory collectives (orl_peer_open)
    when every rank can map the others' exchange buffers, checked against the NCCL
    all-gather path on warm-up steps (statistics must be bit-identical)."""
    from paper_2405_11143_b200.pipeline import run_iteration

    ctx, world, dist, dev = env["ctx"], env["world"], env["dist"], env["dev"]
    if world == 1:
        return "local"
    if env["shared"]:
        ctx.enable_peer()
        return "peer (shared-GPU functional test: no NCCL reference)"
    if args.collective != "peer":
        return "nccl"

    def step():
        return run_iteration(ctx, W["batch"], W["cfg"], W["bufs"], W["src"], W["mb"], pdl_chain=True)

    why = ""
    try:
        ctx.enable_peer()
        ok = 1.0
    except Exception as exc:  # mapping failed on this rank
        ok, why = 0.0, str(exc)[:80]
    t = torch.tensor([ok], device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if t.item() == 1.0:
        try:
            ctx.set_collective("nccl")
            _, st_nccl = step()
            ctx.set_collective("peer")
            _, st_peer = step()
            same = 1.0 if st_nccl == st_peer else 0.0
            why = "" if same else "peer stats differed from NCCL"
        except Exception as exc:
            same, why = 0.0, str(exc)[:80]
        t = torch.tensor([same], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
    if t.item() == 1.0:
        return "peer (single-kernel C1/C2 over peer memory; stats bit-identical to NCCL in warm-up)"
    ctx.set_collective("nccl")
    return f"nccl ({why or 'peer path unavailable on another rank'})"


def run_ours(args):
    env = setup_env(args)
    ctx, world, rank = env["ctx"], env["world"], env["rank"]
    t_start = time.perf_counter()
    W = make_workload(args.config, args, env, args.lengths, args.scaling, args.batch)
    coll = choose_collective(args, env, W)
    R = timed_steps(ctx, W, env, args.steps, args.warmup, pdl_chain=bool(args.pdl_chain))
    value = R["total_tokens"] / (R["ms"] / 1e3)
    roof, stage_ms = roofline(W, R)
    status, st = R["status"], R["stats"]

    # ---- e2e: pinned host buffers, H2D/D2H inside the timed region -----------------
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, env, W, R)

    # ---- oracle on the host cores (rank 0, N = 1 only) ------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = run_cpu_baseline(args, W, value, R["total_tokens"])

    line = None
    if rank == 0:
        c = W["c"]
        line = {"metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": round(R["ms"], 4), "stage_ms_per_step": stage_ms,
                "ms_per_step_stats": {"mean": round(statistics.mean(R["per_step"]), 4),
                                      "median": round(statistics.median(R["per_step"]), 4),
                                      "min": round(min(R["per_step"]), 4), "max": round(max(R["per_step"]), 4),
                                      "rank": "rank 0 (value uses the max over ranks of the mean)"},
                "higher_is_better": True, "scaling": args.scaling if world > 1 else "weak",
                "vs_baseline": None, "dtype": c["dtype"], "data": "synthetic",
                "config": {"workload": _workload_desc(args.config, c, W), "global_batch": W["B_global"],
                           "seq_len": W["T"], "vocab": W["V"], "parallelism": f"dp{world}", "collective": coll,
                           "l2": "inputs larger than L2 (3 x %.1f GB of logits read per step per rank vs 126 MB L2)"
                                 % (W["step_bytes"] / 3 / 1e9),
                           "logits": (f"pool of {W['pool']} micro-batch buffers per model reused across the "
                                      f"{W['n_mb']} micro-batches (the batch does not fit in HBM)")
                           if W["pool"] else "resident",
                           "shards": W["bounds"], "tokens_per_step": R["total_tokens"],
                           "pdl_chain": bool(args.pdl_chain)},
                "status": status, "stats": _stats_round(st), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "clocks": R["clocks"], "gpu_launches": int(R["launches"]),
                "gpu_launches_note": "liborl kernels per timed step (x steps inside the timed region)",
                "gpu_launches_timed_region": int(R["launches"]) * args.steps,
                "per_gpu_tokens_per_s": round(value / world, 1), "per_rank": R["per_rank"],
                "nccl_comm_ranks": world if (env["dist_mode"] and not env["shared"]) else 0}
        if env["shared"]:
            line["test_mode"] = "ORL_BENCH_SHARED_GPU: all ranks on one GPU (functional test, not a measurement)"
    free_workload(W)

    # ---- legs: the other shapes, NEXT-1 / NEXT-4 / graph replay (N = 1 only) ------------
    legs = {}
    if world == 1 and args.legs:
        for spec in args.legs.split(","):
            name, _, lm = spec.partition(":")
            try:
                legs[spec] = run_leg(args, env, name, lm or "full")
            except Exception as exc:  # a leg never hides the headline line
                legs[spec] = {"error": f"{type(exc).__name__}: {str(exc)[:200]}"}
                torch.cuda.empty_cache()
    if rank == 0:
        line["legs"] = legs
        line["wall_s"] = round(time.perf_counter() - t_start, 1)
        print(json.dumps(line), flush=True)
    ctx.close()
    if env["dist_mode"]:
        env["dist"].destroy_process_group()


def run_leg(args, env, name, lengths):
    """A shorter measurement of another shape on one GPU: tokens/s and K1's roofline; the
    full-length llama8b leg adds the CUDA-graph replay, NEXT-1 and NEXT-4."""
    ctx = env["ctx"]
    W = make_workload(name, args, env, lengths, "strong", 0)
    R = timed_steps(ctx, W, env, args.leg_steps, 3)
    roof, stage_ms = roofline(W, R)
    out = {"workload": _workload_desc(name, W["c"], W), "value": round(R["total_tokens"] / (R["ms"] / 1e3), 1),
           "unit": UNIT, "ms_per_step": round(R["ms"], 4), "tokens_per_step": R["total_tokens"],
           "steps": args.leg_steps, "status": R["status"], "roofline": roof, "stage_ms_per_step": stage_ms,
           "clocks": R["clocks"], "gpu_launches": int(R["launches"]),
           "stats": {k: round(R["stats"][k], 6) for k in ("policy_loss", "entropy", "clip_frac", "kl")}}
    if name == "llama8b" and W["lengths"] == "full" and not W["pool"]:
        if args.graph:
            out["graph_replay"] = run_graph(args, ctx, W, R)
        if not args.no_next1:
            out["next1_logits_grad"] = run_next1(args, ctx, W)
        if args.next4:
            out["next4_lmhead"] = run_next4(args, ctx, W)
    free_workload(W)
    return out


def run_cpu_baseline(args, W, value, total_tokens):
    from paper_2405_11143_b200 import synth

    cores = len(os.sched_getaffinity(0))
    c, batch, src, T = W["c"], W["batch"], W["src"], W["T"]
    G = max(1, c["group_size"])

    def sample(n_want, tok_cap, ncores):
        """Whole groups of the first sequences, lengths capped so the sample holds
        about tok_cap valid tokens (the oracle's per-token cost is the 3 V-long rows)."""
        n = max(G, (n_want // G) * G)
        n = min(n, W["mb"]) if W["pool"] else n
        n = max(G, (n // G) * G)
        bnp = {k: v[:n].detach().cpu().numpy() for k, v in batch.items()}
        cap = max(1, -(-tok_cap // n))
        bnp["lengths"] = np.minimum(bnp["lengths"], cap).astype(np.int32)
        hl = {r: synth.to_numpy_logits(src(r, 0, n)[:, :min(cap, T)]) for r in synth.ROLES}
        sh = dict(bnp)
        sh["tokens"] = sh["tokens"][:, :min(cap, T)]
        sh["values_old"] = sh["values_old"][:, :min(cap, T)]
        sh["values_new"] = sh["values_new"][:, :min(cap, T)]
        toks, dt = _oracle_sample(lambda role, k: hl[role][:k], sh, c, n, ncores)
        desc = (f"first {n} sequences ({n // G} whole group(s)) of the same rollout, lengths capped at "
                f"{min(cap, T)} ({toks} tokens, 3 x {toks} vocab rows of V={W['V']}), {dt:.1f} s wall")
        return toks / dt, desc

    v_all, d_all = sample(args.ref_seqs, args.ref_seqs * min(T, 1024), cores)
    cpu = {"value": v_all, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": d_all,
           "cpu_model": _cpu_model()}
    v_one, d_one = sample(1, 1024, 1)            # the same oracle on one core
    cpu["single_core"] = {"value": v_one, "unit": UNIT, "cores": 1, "sample": d_one}
    cpu["extrapolated_step_s"] = round(total_tokens / v_all, 1)
    cpu["gpu_over_cpu"] = round(value / v_all, 1)
    return cpu


def run_graph(args, ctx, W, R_eager):
    """The timed step (all S1..S10 launches, C1/C2 included) captured once as a CUDA
    graph (pipeline.GraphStep, orl_finalize_async) and replayed K times; the replayed
    statistics must equal the eager step's bit for bit."""
    from paper_2405_11143_b200.pipeline import GraphStep

    step = GraphStep(ctx, W["batch"], W["cfg"], W["bufs"], W["src"], W["mb"], pdl_chain=True)
    gs = torch.cuda.current_stream()
    for _ in range(2):
        step.replay()
    torch.cuda.synchronize()
    same = step.result() == (R_eager["status"], R_eager["stats"])
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(gs)
    for _ in range(args.leg_steps):
        step.replay()
    b.record(gs)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.leg_steps
    return {"tokens_per_s": round(W["n_tok"] / (ms / 1e3), 1), "ms_per_step": round(ms, 4),
            "kernels_per_graph": int(step.kernels), "graph_launches_per_step": 1,
            "stats_bit_identical_to_eager": bool(same), "steps": args.leg_steps}


def run_next1(args, ctx, W):
    """Time the NEXT-1 backward pass (orl_logits_grad, K5) over every micro-batch of the
    actor logits (reads V*2 B and writes V*2 B per token), and the fused actor pass
    (orl_ppo_loss_and_grad: loss epilogue + backward in one pass, the row re-read from L2)."""
    from paper_2405_11143_b200 import orl

    batch, cfg, bufs, logits, mb = W["batch"], W["cfg"], W["bufs"], W["logits"], W["mb"]
    B, T, V = W["B_rank"], W["T"], W["V"]
    n_tok = W["n_tok"]
    free = torch.cuda.mem_get_info()[0]
    need = B * T * V * 2
    if need > free - (4 << 30):
        return {"skipped": f"needs {need / 1e9:.1f} GB for dlogits"}
    dl = torch.empty(B, T, V, dtype=logits["new"].dtype, device=W["bufs"].adv.device)
    tok, L = batch["tokens"], batch["lengths"]
    stream = torch.cuda.current_stream()

    def once():
        for s in range(0, B, mb):
            e = min(B, s + mb)
            orl.orl_logits_grad(ctx, tok, L, logits["new"][s:e], cfg.ppo, bufs.lse, bufs.entropy, bufs.dlogp,
                                dl[s:e], seq_offset=s, inv_temp=cfg.inv_temp, stream=stream)

    def fused():
        critic = cfg.critic
        for s in range(0, B, mb):
            e = min(B, s + mb)
            orl.orl_ppo_loss_and_grad(ctx, tok, L, logits["new"][s:e], cfg.ppo, bufs.logp_old, bufs.adv,
                                      bufs.logp_new, seq_offset=s, inv_temp=cfg.inv_temp, logp_ref=bufs.logp_ref,
                                      ret=bufs.ret if critic else None,
                                      v_new=batch["values_new"] if critic else None,
                                      v_old=batch["values_old"] if critic else None, entropy=bufs.entropy,
                                      lse=bufs.lse, dloss_dlogp=bufs.dlogp, dloss_dv=bufs.dv if critic else None,
                                      flags=bufs.flags, adv_lo=bufs.adv_lo, dlogits=dl[s:e], stream=stream)

    def timed(fn):
        for _ in range(2):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    reps = max(10, args.leg_steps)       # each rep = every micro-batch of the actor logits (~12 ms)
    prev = ctx.pdl_chain
    ctx.pdl_chain = True
    ms = timed(once)
    byts = n_tok * V * 2 * 2
    peak, _ = _peaks()
    ms_f = timed(fused)
    ctx.pdl_chain = prev
    del dl
    torch.cuda.empty_cache()
    ach_f = byts / (ms_f / 1e3) / 1e9
    return {"tokens_per_s": round(n_tok / (ms / 1e3), 1), "ms_per_pass": round(ms, 4),
            "roofline": {"bound": "hbm", "achieved": round(byts / (ms / 1e3) / 1e9, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(byts / (ms / 1e3) / 1e9 / peak, 4),
                         "bytes": "V*2 read + V*2 written per valid token"},
            "kernel": "k5_tma_kernel", "launches": len(range(0, B, mb)), "reps": reps,
            "fused_actor_pass": {"api": "orl_ppo_loss_and_grad", "tokens_per_s": round(n_tok / (ms_f / 1e3), 1),
                                 "ms": round(ms_f, 4), "algorithmic_GBps": round(ach_f, 1),
                                 "frac": round(ach_f / peak, 4),
                                 "bytes": "V*2 read + V*2 written per valid token (the L2 re-read is not counted)"}}


def run_next4(args, ctx, W):
    """NEXT-4 leg (not part of `value`): the whole iteration with every S1 pass computed
    from the model's final hidden states through its LM head, [R, d] x [V, d]^T on the
    tcgen05 tensor cores fused with the online log-sum-exp (K6, orl_lmhead_*), against
    the unfused baseline: cuBLAS bf16 GEMM (torch.matmul) writing each micro-batch's
    logits to HBM, then K1.  d = 4096 (Llama-3-8B hidden size)."""
    from paper_2405_11143_b200 import synth
    from paper_2405_11143_b200.pipeline import LmHeadRows, run_iteration

    batch, cfg, bufs, mb = W["batch"], W["cfg"], W["bufs"], W["mb"]
    B, T, V, d = W["B_rank"], W["T"], W["V"], args.hidden
    dev = bufs.adv.device
    n_tok = W["n_tok"]
    stream = torch.cuda.current_stream()
    # the leg's logits are no longer needed: free them for the hidden states + W
    W["logits"].clear()
    torch.cuda.empty_cache()
    R = B * T
    g = torch.Generator(device=dev).manual_seed(synth.role_seed(4321, 30_000, 0))
    # as synth.make_lmhead_batch: hidden_old = s_r N(0, I), ref = old + 0.05 N, new = old + 0.03 N
    hid = {r: torch.empty(R, d, dtype=torch.bfloat16, device=dev) for r in synth.ROLES}
    for s in range(0, R, 16384):
        e = min(R, s + 16384)
        base = torch.randn(e - s, d, generator=g, device=dev) * (torch.rand(e - s, 1, generator=g, device=dev) + 0.5)
        for r, sd in zip(synth.ROLES, (0.0, 0.05, 0.03)):
            hid[r][s:e] = (base + sd * torch.randn(e - s, d, generator=g, device=dev)).to(torch.bfloat16)
    Wt = torch.empty(V, d, dtype=torch.bfloat16, device=dev)
    for s in range(0, V, 8192):
        e = min(V, s + 8192)
        Wt[s:e] = (torch.randn(e - s, d, generator=g, device=dev) * (3.0 / d ** 0.5)).to(torch.bfloat16)
    fused_src = lambda role, s, e: LmHeadRows(hid[role][s * T:e * T], Wt)  # noqa: E731
    scratch = torch.empty(mb * T, V, dtype=torch.bfloat16, device=dev)

    def unfused_src(role, s, e):
        out = scratch[: (e - s) * T]
        torch.matmul(hid[role][s * T:e * T], Wt.t(), out=out)
        return out.view(e - s, T, V)

    def timed(src, reps, chain):
        for _ in range(2):
            run_iteration(ctx, batch, cfg, bufs, src, mb, stream=stream, pdl_chain=chain)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            status, st = run_iteration(ctx, batch, cfg, bufs, src, mb, stream=stream, pdl_chain=chain)
        b.record(stream)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps, status, st

    reps = max(2, args.leg_steps // 3)
    l0 = ctx.launch_count
    ms_f, status, st = timed(fused_src, reps, True)
    launches = (ctx.launch_count - l0) // (reps + 2)
    # cuBLAS writes the logits right before each K1: K1 must wait for it (no PDL chaining)
    ms_u, status_u, st_u = timed(unfused_src, reps, False)
    flops = 3 * 2.0 * R * d * V
    peak, peak_src = _bf16_peak(sustained=True)
    ach = flops / (ms_f / 1e3) / 1e12
    del scratch
    # end to end from the host: each micro-batch's hidden states (the inputs of this path; the
    # LM-head weight stays resident like the model's other weights) copied from pinned host
    # memory on a copy stream, double-buffered, inside the timed region
    host = {r: hid[r].cpu().pin_memory() for r in synth.ROLES}
    stage = [{r: torch.empty(mb * T, d, dtype=torch.bfloat16, device=dev) for r in synth.ROLES} for _ in range(2)]
    copy = torch.cuda.Stream()
    order = [(r, s0) for r in ("old", "ref", "new") for s0 in range(0, B, mb)]

    def e2e_step():
        pending, slot_free, cnt = {}, [None, None], {"i": 0}

        def fetch(i):
            r, s0 = order[i]
            e0 = min(B, s0 + mb)
            with torch.cuda.stream(copy):
                if slot_free[i % 2] is not None:
                    copy.wait_event(slot_free[i % 2])
                stage[i % 2][r][: (e0 - s0) * T].copy_(host[r][s0 * T:e0 * T], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
            pending[i] = ev

        def src(role, s0, e0):
            i = cnt["i"]
            cnt["i"] += 1
            stream.wait_event(pending.pop(i))
            if i + 1 < len(order):
                fetch(i + 1)
            return LmHeadRows(stage[i % 2][role][: (e0 - s0) * T], Wt)

        def hook(tag):
            def after():
                ev = torch.cuda.Event()
                ev.record(stream)
                slot_free[(cnt["i"] - 1) % 2] = ev
            return after

        fetch(0)
        return run_iteration(ctx, batch, cfg, bufs, src, mb, stream=stream, on_k1=hook, pdl_chain=False)

    e2e_step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        status_e, st_e = e2e_step()
    torch.cuda.synchronize()
    ms_e = (time.perf_counter() - t0) / reps * 1e3
    h2d = 3 * R * d * 2 + sum(v.numel() * v.element_size() for v in batch.values())
    e2e = {"value": round(n_tok / (ms_e / 1e3), 1), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": 16 * 8 + 4 * 8, "ms_per_step": round(ms_e, 3), "status": status_e,
           "stats_bit_identical_to_device_step": bool((status_e, st_e) == (status, st)),
           "note": "hidden states of the three models streamed from pinned host memory each step "
                   "(double-buffered copy stream; the per-token inputs stay resident); host clock"}
    del host, stage, hid, Wt
    torch.cuda.empty_cache()
    return {"tokens_per_s": round(n_tok / (ms_f / 1e3), 1), "ms_per_step": round(ms_f, 3), "status": status,
            "hidden": d, "reps": reps, "gpu_launches": int(launches),
            "policy_loss": round(st["policy_loss"], 6), "entropy": round(st["entropy"], 6),
            "roofline": {"bound": "tensor", "achieved": round(ach, 1), "peak": peak, "unit": "TFLOP/s",
                         "frac": round(ach / peak, 4), "flops": "3 x 2 R d V per step (old, ref, actor heads)",
                         "peak_source": peak_src, "kernel": "k6_lmhead_2sm_kernel + k6_merge_kernel (whole step)"},
            "unfused_cublas_plus_k1": {"tokens_per_s": round(n_tok / (ms_u / 1e3), 1), "ms_per_step": round(ms_u, 3),
                                       "status": status_u, "policy_loss": round(st_u["policy_loss"], 6)},
            "speedup_vs_unfused": round(ms_u / ms_f, 4), "e2e": e2e}


def run_e2e(args, env, W, R_dev):
    """The same iteration end to end through the public API with the step's inputs in
    pinned HOST memory.  Every step copies, host -> device, each micro-batch's own logits
    of the three models (double-buffered on a copy stream, overlapping the kernels) and the
    per-token inputs, and orl_finalize reads the statistics back (D2H) and synchronises.
    Host logits: a pinned copy of each micro-batch buffer the device step reads (the pool
    slots for a pooled config, else the micro-batches themselves up to ~48 GB; micro-batch
    k is then slot k mod H).  The e2e statistics are checked bit for bit against a
    device-resident step that reads the same micro-batch buffers."""
    from paper_2405_11143_b200.pipeline import run_iteration

    dist, dev, ctx, world = env["dist"], env["dev"], env["ctx"], env["world"]
    batch, cfg, bufs, mb, T, V = W["batch"], W["cfg"], W["bufs"], W["mb"], W["T"], W["V"]
    B = W["B_rank"]
    logits = W["logits"]
    mb_bytes = 3 * mb * T * V * W["elt"]
    # pinned host memory: at most ~56 GB per node (2 grpo buffers per model), split over its ranks
    budget = 56e9 / (world if world > 1 else 1)
    H = min(W["pool"], max(1, int(budget // mb_bytes))) if W["pool"] else max(1, min(W["n_mb"], int(budget // mb_bytes)))
    try:
        import psutil
        avail = psutil.virtual_memory().available
    except Exception:  # pragma: no cover
        avail = None
    ok = avail is None or H * mb_bytes * world <= 0.6 * avail
    # device staging (2 micro-batch slots x 3 models); with ORL_BENCH_SHARED_GPU every rank's
    # copy lives on the one GPU
    dev_need = 2 * mb_bytes * (world if env["shared"] else 1)
    dev_ok = torch.cuda.mem_get_info(dev)[0] >= 1.1 * dev_need
    ok = ok and dev_ok
    if env["dist_mode"]:                      # every rank takes the same decision
        t = torch.tensor([1.0 if ok else 0.0], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        ok = t.item() == 1.0
    if not ok:
        if not dev_ok:
            return {"skipped": f"needs {dev_need / 1e9:.0f} GB of free device memory for the staging slots"}
        return {"skipped": f"needs {H * mb_bytes * world / 1e9:.0f} GB of pinned host memory "
                           f"({(avail or 0) / 1e9:.0f} GB available on this node)"}
    # device view of slot h: pool slot h, or the resident micro-batch h
    dev_slot = {r: [logits[r][h * mb:h * mb + mb] for h in range(H)] for r in logits}
    host = {r: [torch.empty(x.shape, dtype=x.dtype, pin_memory=True).copy_(x) for x in dev_slot[r]] for r in logits}
    small = {k: v.cpu().pin_memory() for k, v in batch.items()}
    stage = [{r: torch.empty_like(dev_slot[r][0]) for r in logits} for _ in range(2)]
    dbatch = {k: torch.empty_like(v) for k, v in batch.items()}
    comp, copy = torch.cuda.current_stream(), torch.cuda.Stream()
    order = [(r, s) for r in ("old", "ref", "new") for s in range(0, B, mb)]
    h2d = sum(v.numel() * v.element_size() for v in small.values())
    h2d += sum((min(B, s + mb) - s) * T * V * W["elt"] for r, s in order)
    d2h = 16 * 8 + 4 * 8

    def one_step():
        for k, v in small.items():
            dbatch[k].copy_(v, non_blocking=True)
        slot_free = [None, None]
        pending = {}
        counter = {"i": 0}

        def fetch(i):
            r, s = order[i]
            e = min(B, s + mb)
            with torch.cuda.stream(copy):
                if slot_free[i % 2] is not None:
                    copy.wait_event(slot_free[i % 2])
                stage[i % 2][r][: e - s].copy_(host[r][(s // mb) % H][: e - s], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
            pending[i] = ev

        def src(role, s, e):
            i = counter["i"]
            counter["i"] += 1
            comp.wait_event(pending.pop(i))
            if i + 1 < len(order):
                fetch(i + 1)
            return stage[i % 2][role][: e - s]

        def hook(tag):
            def after():
                i = counter["i"] - 1
                ev = torch.cuda.Event()
                ev.record(comp)
                slot_free[i % 2] = ev          # slot i%2 may be refilled after this K1
            return after

        fetch(0)
        # the logits arrive by copies on another stream: no PDL chaining (every K1 waits)
        return run_iteration(ctx, dbatch, cfg, bufs, src, mb, stream=comp, on_k1=hook, pdl_chain=False)

    big = W["step_bytes"] > 2e11
    steps = args.e2e_steps or (1 if big else max(2, args.steps // 5))
    if not big:
        one_step()                                      # warm-up (copy stream, pinned paths)
    torch.cuda.synchronize()
    if env["dist_mode"]:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        status, st = one_step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    if env["dist_mode"]:
        tt = torch.tensor([dt], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    # the device-resident step over the same micro-batch buffers gives the same bits (run on
    # every rank: the statistics are global, and the collectives need every rank)
    ref_status, ref_st = run_iteration(ctx, batch, cfg, bufs, lambda r, s, e: dev_slot[r][(s // mb) % H][: e - s],
                                       mb, pdl_chain=True)
    same = (status, st) == (ref_status, ref_st)
    del stage, host
    torch.cuda.empty_cache()
    total = R_dev["total_tokens"]
    return {"value": round(total / dt, 1), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": d2h, "steps": steps, "status": status,
            "stats_bit_identical_to_device_step": bool(same),
            "host_logits": f"{H} pinned micro-batch buffer(s) per model ({H * mb_bytes / 1e9:.1f} GB); "
                           f"micro-batch k streams buffer k mod {H}",
            "note": "logits streamed from pinned host memory over PCIe each step (double-buffered); host clock"}


# ----------------------------------------------------------------------------- launcher
def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=10,
                    help="untimed steps; default 10: the paper excludes the first 10 steps (P:94, S:535)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="grpo", help="BASELINE.json config: tiny, llama8b, longcot, grpo, rpp8")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: split the config's batch over the ranks (strong) or give each rank one (weak)")
    ap.add_argument("--lengths", default="full", choices=["full", "secondary"],
                    help="full: every L_b = T; secondary: SURVEY 8(d) ragged lengths")
    ap.add_argument("--batch", type=int, default=0, help="override B (testing)")
    ap.add_argument("--pool", type=int, default=2, help="micro-batch buffers per model when the batch does not fit")
    ap.add_argument("--legs", default=LEGS_DEFAULT, help="comma list of config[:secondary] legs ('' = none)")
    ap.add_argument("--leg-steps", type=int, default=10)
    ap.add_argument("--ref-seqs", type=int, default=4, help="oracle sample size (sequences)")
    ap.add_argument("--e2e-steps", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-next1", action="store_true")
    ap.add_argument("--next4", type=int, default=1, help="run the NEXT-4 LM-head leg (1/0)")
    ap.add_argument("--collective", default="peer", choices=["peer", "nccl"],
                    help="C1/C2 transport at N > 1 (peer: single peer-memory kernels, NCCL-checked)")
    ap.add_argument("--hidden", type=int, default=4096, help="NEXT-4 hidden size d")
    ap.add_argument("--graph", type=int, default=1, help="time the CUDA-graph replay of the llama8b leg (1/0)")
    ap.add_argument("--pdl-chain", type=int, default=1,
                    help="headline: K1 launches overlap the previous launch's tail (orl_set_pdl_chain; the logits "
                         "are resident, nothing else writes them)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run on this node
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", f"--master-port={_free_port()}", os.path.abspath(__file__),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
