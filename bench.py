#!/usr/bin/env python
"""Benchmark of the HOLMES serving hot path on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], "c2"): a 4-member ResNet1D ensemble
(ecg-i-w32-d8, ecg-i-w64-d4, ecg-ii-w32-d8, ecg-iii-w32-d8 of the paper's
60-member zoo) serving 64 beds x 3 ECG leads at 250 Hz; every 1 s tick each
bed's latest 7500-sample window is z-normalised and scored by every member and
the member sigmoids are averaged.  One *step* = one tick over all beds.
Synthetic seeded ECG streams (`synth.ecg_block`), random-init synthetic
weights (no checkpoints).

  value   : patient-windows/s over all ranks, inputs already in HBM, device
            time (CUDA events per step on the serving stream, L2 flushed by a
            256 MiB write between steps), max over ranks.
  latency : device tick p50/p95/p99 (nearest rank, runtime.py:246) and the
            host-timed per-tick END-TO-END p50/p95/p99 of one blocking
            `EnsembleEngine.tick` (pinned H2D of the hop + D2H of the scores).
  e2e     : the same metric through the public API with host buffers (H2D of
            each tick's samples + D2H of its scores inside the timed region),
            host wall clock, max over ranks: `EnsembleEngine.submit/collect`
            (tick t+1 enqueued before tick t is collected).
  parity  : the last timed tick's outputs vs the CPU oracle
            (oracle/cpu_path.cpu_tick, fp32) on sampled beds.
  roofline: the polyphase tcgen05 conv kernel K4b (the dominant kernel) —
            algorithmic conv FLOPs / its event-timed launch durations (one
            eager tick on the serving stream, an event after every launch);
            peak = MEASURED_PEAKS.json dense 16-bit burst TFLOP/s (the
            sustained fraction is reported beside it).
  cpu_baseline: the CPU oracle port of the same 64-bed tick (PyTorch fp32, all
            host threads), rank 0 at N=1, repeated for ~10 s.

Multi-GPU (`--gpus N`; re-executes itself under torch.distributed.run when
WORLD_SIZE is unset; refuses when N exceeds the visible devices):
  --mode patient (default): each rank serves its own 64 beds (the reference's
      units are independent: no collective on the data path), "weak" scaling.
  --mode member (config c5): the selected members are FLOP-balanced over the
      ranks, every rank serves all beds, and one NCCL reduce of the per-bed
      partial sums [2, P] per tick combines them (timed with events);
      "strong" scaling.
`--impl reference` times the CPU oracle port of the same tick on the host
cores (the reference has no CNN and no GPU path; its scorer is an analytic
stand-in), rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "patient-windows/sec/GPU (250 Hz ECG, 64-bed); p99 tick latency vs 200 ms SLO"
UNIT = "patient-windows/s"
MEMBERS = [10, 13, 30, 50]
SLO_MS = 200.0
W = 7500


def parse(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)  # >= 1000 ticks per config
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--mode", default="patient", choices=["patient", "member"])
    ap.add_argument("--members", default="c2", choices=["c2", "all"], help="c2 ensemble or the whole 60-zoo")
    ap.add_argument("--patients", type=int, default=64, help="beds per GPU (patient mode) / in total (member mode)")
    ap.add_argument("--hop", type=int, default=250)
    ap.add_argument("--parity-beds", type=int, default=8)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu (no clocks / cpu / extras)")
    ap.add_argument("--no-extras", action="store_true", help="skip the 1024-bed, c3 and profiler-sweep side measurements")
    ap.add_argument("--ref-budget-s", type=float, default=150.0, help="reference arm: cap on the timed CPU seconds")
    return ap.parse_args(argv)


# ------------------------------------------------------------------ launcher / ranks
def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def launch_argv(args_list, gpus: int, port: int) -> list:
    """The torch.distributed.run command line that re-executes this bench with one rank per GPU."""
    return [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={gpus}",
            "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + list(args_list)


def rank_env(env=None) -> tuple[int, int, int]:
    env = os.environ if env is None else env
    return int(env.get("RANK", "0")), int(env.get("WORLD_SIZE", "1")), int(env.get("LOCAL_RANK", "0"))


def check_world(args, env=None, visible=None):
    """None when the launch is consistent, else the reason to refuse."""
    rank, world, local = rank_env(env)
    if world != args.gpus:
        return f"--gpus {args.gpus} but WORLD_SIZE={world}"
    if visible is not None and visible < args.gpus:
        return f"--gpus {args.gpus} but only {visible} CUDA device(s) are visible"
    if args.mode == "member" and args.impl == "b200":
        n = 60 if args.members == "all" else len(MEMBERS)
        if n < world:
            return f"member mode: {n} members cannot be spread over {world} ranks"
    return None


class Ranks:
    """Max/sum over ranks (NCCL on GPUs, gloo on CPU tensors) and the barrier; world 1 is local."""

    def __init__(self, world: int, device=None):
        self.world = world
        self.device = device

    def _red(self, x: float, op):
        if self.world == 1:
            return float(x)
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(x)], dtype=torch.float64, device=self.device)
        dist.all_reduce(t, op=op)
        return float(t.item())

    def max(self, x: float) -> float:
        import torch.distributed as dist
        return self._red(x, dist.ReduceOp.MAX if self.world > 1 else None)

    def sum(self, x: float) -> float:
        import torch.distributed as dist
        return self._red(x, dist.ReduceOp.SUM if self.world > 1 else None)

    def barrier(self):
        if self.world > 1:
            import torch.distributed as dist
            dist.barrier()


def workload(args, world: int) -> dict:
    members = (["ecg-i-w32-d8", "ecg-i-w64-d4", "ecg-ii-w32-d8", "ecg-iii-w32-d8"] if args.members == "c2"
               else ["the whole 60-member zoo"])
    if args.mode == "patient":
        name = ("c2: 4-member ResNet1D ensemble" if args.members == "c2" else "c3: 60-member zoo") + \
            f", {args.patients}-bed 250 Hz 3-lead ECG per GPU, 7500-sample sliding window, 1 s tick"
        par = f"patient-sharded x{world}"
    else:
        name = ("c5: " if args.members == "all" else "") + \
            f"member-sharded ensemble over {args.patients} beds, 250 Hz 3-lead ECG, 7500-sample window, 1 s tick"
        par = f"member-sharded x{world} (NCCL reduce of per-bed partial sums per tick)"
    return {
        "workload": name,
        "members": members,
        "patients_per_gpu": args.patients if args.mode == "patient" else None,
        "patients_total": args.patients * world if args.mode == "patient" else args.patients,
        "window": W,
        "hop": args.hop,
        "aggregation": "mean of member sigmoids (+ mean latent)",
        "precision": "fp16 operands, fp32 accumulate; fp16 activations",
        "l2": "flushed between timed steps (256 MiB device write)",
        "parallelism": par,
    }


# ------------------------------------------------------------------ measurement helpers
class Clocks:
    """nvidia-smi sampler running during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "20", "-i", str(index)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.p = None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        out, _ = self.p.communicate(timeout=10)
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                smax = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def peaks():
    """(burst TF/s, sustained TF/s, HBM GB/s, source)."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return (float(d["bf16_tflops"]), float(d["bf16_tflops_sustained"]), float(d["hbm_gbs"]),
                "measured (MEASURED_PEAKS.json)")
    except (OSError, KeyError, ValueError):
        return 1640.0, 1400.0, 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic():
    path = os.path.join(ROOT, "profiles", "ncu_conv_summary.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return d.get("dram_bytes_per_launch"), d
    except (OSError, ValueError):
        return None, None


def pct(v, q):
    s = sorted(v)
    return s[max(0, int(np.ceil(q / 100 * len(s))) - 1)]  # nearest rank, as runtime.py:246


def lat(v) -> dict:
    return {"p50": pct(v, 50), "p95": pct(v, 95), "p99": pct(v, 99), "max": max(v), "n": len(v)}


def selection(args):
    from paper_2008_04063_b200.zoo import Selector, holmes_zoo
    zoo = holmes_zoo()
    return zoo, (Selector.from_indices(60, MEMBERS) if args.members == "c2" else Selector.ones(60))


def sample_beds(P: int, n: int) -> list:
    return sorted(set(np.linspace(0, P - 1, max(1, min(n, P))).astype(int).tolist()))


def streams_for(pids, hop: int, ticks: int, seed: int = 0) -> np.ndarray:
    """Seeded synthetic ECG [P, 3, W - hop + ticks*hop]: the prefill, then one hop per tick."""
    from paper_2008_04063_b200 import synth
    return synth.ecg_block(seed, pids, 3, 0, W - hop + ticks * hop)


def parity_check(zoo, sel, streams, end, beds, ml, prob, mean_logit) -> dict:
    """Oracle (CPU fp32) vs the device outputs of the tick that ended at sample `end`."""
    from oracle import cnn, cpu_path
    oml, oprob, omean = cpu_path.cpu_tick(zoo, sel, streams, end, beds=beds)
    dl = float(np.abs(ml[beds] - oml).max())
    dp = float(max(np.abs(prob[beds] - oprob).max(), np.abs(cnn.sigmoid(ml[beds]) - cnn.sigmoid(oml)).max()))
    dm = float(np.abs(mean_logit[beds] - omean).max())
    return {"beds": len(beds), "bed_ids": beds, "max_dprob": dp, "max_dlogit": dl, "max_dmean_logit": dm,
            "tol": {"prob": 1e-3, "logit": 2e-2}, "ok": bool(dp <= 1e-3 and dl <= 2e-2 and dm <= 2e-2),
            "oracle": "oracle/cpu_path.cpu_tick (PyTorch fp32 CPU, the oracle's own layer table)"}


def device_outputs(eng, P: int, M: int):
    import torch

    from paper_2008_04063_b200.parallel import CudaView
    ml, ep, el = eng.device_outputs()
    torch.cuda.synchronize()
    t = lambda p, shape: torch.as_tensor(CudaView(p, shape), device="cuda").cpu().numpy().copy()  # noqa: E731
    return t(ml, (P, M)), t(ep, (P,)), t(el, (P,))


def cpu_baseline(zoo, sel, P, hop, budget_s=10.0, seed=0):
    """The CPU oracle port of the same P-bed tick, repeated for about budget_s seconds (>= 1 tick)."""
    import torch

    from oracle.cpu_path import cpu_tick, params_for
    torch.set_num_threads(os.cpu_count() or 1)
    for i in sel.indices():
        params_for(zoo.profiles[i], seed)
    streams = streams_for(P, hop, 8, seed)
    end = W
    cpu_tick(zoo, sel, streams[:1], end, seed=seed)  # warm
    n, t0 = 0, time.perf_counter()
    while True:
        cpu_tick(zoo, sel, streams, end, seed=seed)
        n += 1
        end = min(end + hop, streams.shape[2])
        dt = time.perf_counter() - t0
        if dt >= budget_s or n >= 8:
            break
    return {"value": P * n / dt, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "port",
            "sample": f"{n} full {P}-bed ticks x {sel.popcount} members, PyTorch fp32 CPU oracle, {dt:.1f} s"}


def tick_roofline(zoo, sel, P, peak_tf, peak_gbs):
    """Tick roofline time: sum over every layer of max(FLOPs / tensor peak, algorithmic
    bytes / HBM peak) — input + output (+ shortcut) activations in fp16, per window."""
    from paper_2008_04063_b200 import arch
    t = f_tot = b_tot = 0.0
    for i in sel.indices():
        pr = zoo.profiles[i]
        for L in arch.member_layers(pr.width, pr.depth):
            f = L.flops * P
            b = (L.cin * L.lin + (0 if L.head else L.cout * L.lout) +
                 (L.res_c * L.lin if L.res != "none" else 0)) * 2 * P
            t += max(f / (peak_tf * 1e12), b / (peak_gbs * 1e9))
            f_tot += f
            b_tot += b
    return {"ms": t * 1e3, "flops": f_tot, "bytes": b_tot,
            "def": "sum_layers max(FLOPs/burst tensor peak, (in+out+shortcut) fp16 bytes/HBM peak)"}


def host_tick_latency(eng, blocks, warm=3):
    """Per-tick host-timed end-to-end latency of one blocking EnsembleEngine.tick (pinned H2D of the
    hop + graph + D2H of the scores) in ms, nearest-rank percentiles."""
    import torch

    from paper_2008_04063_b200.engine import TickResult
    P, M = eng.patients, eng.selector.popcount
    out = TickResult(eng.member_ids, torch.empty((P, M), pin_memory=True).numpy(),
                     torch.empty(P, pin_memory=True).numpy(), torch.empty(P, pin_memory=True).numpy())
    for i in range(warm):
        eng.tick(blocks[i % len(blocks)], out=out)
    t = []
    for i in range(len(blocks)):
        t0 = time.perf_counter()
        eng.tick(blocks[i], out=out)
        t.append((time.perf_counter() - t0) * 1e3)
    return lat(t)


def tick_at(zoo, sel, P, hop, device, K=30, warm=5, e2e_ticks=0):
    """Side measurement: the same ensemble at P beds (graph tick, device time, L2 flushed), the
    memory-bound stream kernels' achieved GB/s, and the host-timed e2e per-tick latency."""
    import torch

    from paper_2008_04063_b200.engine import EnsembleEngine
    eng = EnsembleEngine(zoo, sel, P, hop=hop, device=device)
    eng.ingest((np.random.default_rng(1).standard_normal((P, 3, W)) * 0.3).astype(np.float32))
    blk = torch.randn(P, 3, hop, device="cuda") * 0.3
    st = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ms = []
    with torch.cuda.stream(st):
        for i in range(warm + K):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            eng.stage_device(blk.data_ptr(), st.cuda_stream)
            eng.tick_device(st.cuda_stream)
            b.record(st)
            if i >= warm:
                ms.append((a, b))
    torch.cuda.synchronize()
    t = [a.elapsed_time(b) for a, b in ms]
    flops, _ = eng.tick_work()
    kinds, kms, _, kbytes = eng.profile_tick(st.cuda_stream)
    torch.cuda.synchronize()
    stream_k = {}
    for kind, name in ((0, "ingest_window"), (3, "aggregate")):
        sel_k = kinds == kind
        if sel_k.any():
            tms = float(kms[sel_k].sum())
            stream_k[name] = {"ms": tms, "bytes": float(kbytes[sel_k].sum()),
                              "gbs": float(kbytes[sel_k].sum()) / (tms / 1e3) / 1e9 if tms > 0 else None}
    out = {"patients": P, "tick_ms": lat(t), "patient_windows_per_s": P / (float(np.mean(t)) / 1e3),
           "tflops": flops / (float(np.mean(t)) / 1e3) / 1e12, "ticks": K, "stream_kernels_eager": stream_k}
    if e2e_ticks:
        hb = torch.empty((e2e_ticks, P, 3, hop), dtype=torch.float32, pin_memory=True).numpy()
        hb[:] = (np.random.default_rng(2).standard_normal(hb.shape) * 0.3).astype(np.float32)
        out["e2e_tick_ms"] = host_tick_latency(eng, hb)
        out["e2e_tick_ms"]["def"] = "host perf_counter around one blocking EnsembleEngine.tick (pinned H2D + D2H)"
    eng.close()
    return out


def sweep_bench(device):
    """Config c4: exhaustive profiler sweep over N=20000 recorded windows (synthetic cohort),
    n=10 (1023 candidates) and n=16 (65535), K6 on the device; CPU oracle on a bounded sample."""
    from oracle import auc as oauc
    from paper_2008_04063_b200 import cohort as hc
    from paper_2008_04063_b200 import composer
    from paper_2008_04063_b200.zoo import generate_zoo
    out = {}
    for n, grid in ((10, ([8, 16, 32, 64, 128], [2, 4])), (16, ([8, 16, 32, 64], [2, 4, 8, 16]))):
        z = generate_zoo(1, grid[0], grid[1], seed=3)
        coh = hc.synthesize_cohort(z, 10000, 10000, 0.5, 0)
        dev = coh.device(device)
        dev.auc_range(1, 64)                       # warm
        t0 = time.perf_counter()
        aucs = composer.sweep_aucs(coh, device)
        dt = time.perf_counter() - t0
        best = int(np.argmax(aucs)) + 1
        S = (1 << n) - 1
        out[f"n{n}"] = {"candidates": S, "N": 20000, "seconds": dt, "candidates_per_s": S / dt,
                        "best_auc_selector": format(best, f"0{n}b")[::-1], "best_auc": float(aucs[best - 1])}
    # the recording leg of the profiler (north star (4)): every member of the n=10 zoo over
    # N=20000 recorded windows on the serving kernels (tumbling, 1024 windows per device tick)
    z = generate_zoo(1, [8, 16, 32, 64, 128], [2, 4], seed=3)
    rng = np.random.default_rng(5)
    wins = (rng.standard_normal((20000, 1, 7500)) * 0.3).astype(np.float32)
    labels = (rng.random(20000) < 0.5).astype(np.int8)
    hc.record_cohort(z, wins[:2048], labels[:2048], batch=1024, device=device)  # warm (build + graph)
    t0 = time.perf_counter()
    hc.record_cohort(z, wins, labels, batch=1024, device=device)
    dt = time.perf_counter() - t0
    out["record"] = {"windows": 20000, "members": z.n, "seconds": dt, "windows_per_s": 20000 / dt,
                     "member_windows_per_s": 20000 * z.n / dt,
                     "def": "cohort.record_cohort: host windows -> device -> every member's forward -> logits "
                            "(includes engine setup; 1024 windows per tick, pipelined submit/collect)"}
    z = generate_zoo(1, [8, 16, 32, 64, 128], [2, 4], seed=3)
    coh = hc.synthesize_cohort(z, 10000, 10000, 0.5, 0)
    vals = np.arange(1, 65)
    t0 = time.perf_counter()
    oauc.sweep(coh.labels, coh.scores, vals)
    dt = time.perf_counter() - t0
    out["cpu_oracle"] = {"candidates_per_s": len(vals) / dt, "cores": 1, "sample": "64 candidates of n=10, N=20000"}
    return out


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank, world, _ = rank_env()
    if rank != 0:
        return
    import torch

    from oracle.cpu_path import cpu_tick, params_for
    torch.set_num_threads(os.cpu_count() or 1)
    zoo, sel = selection(args)
    for i in sel.indices():
        params_for(zoo.profiles[i])
    P = args.patients if args.mode == "patient" else args.patients
    streams = streams_for(P, args.hop, 4)
    end = W
    cpu_tick(zoo, sel, streams, end)                       # one full tick: its cost sizes the run
    t0 = time.perf_counter()
    cpu_tick(zoo, sel, streams, end)
    per_tick = time.perf_counter() - t0
    # every step is the full P-bed tick unless (steps + warmup) of them would overrun the budget;
    # then each step is a bounded bed sample of it (stated in `sample`)
    beds = P
    if (args.steps + args.warmup) * per_tick > args.ref_budget_s:
        beds = max(1, int(P * args.ref_budget_s / ((args.steps + args.warmup) * per_tick)))
    sub = streams[:beds]
    for k in range(args.warmup):
        cpu_tick(zoo, sel, sub, min(W + (k % 4) * args.hop, streams.shape[2]))
    t = []
    for k in range(args.steps):
        t0 = time.perf_counter()
        cpu_tick(zoo, sel, sub, min(W + (k % 4) * args.hop, streams.shape[2]))
        t.append(time.perf_counter() - t0)
    dt = float(sum(t))
    value = beds * args.steps / dt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak" if args.mode == "patient" else "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded ECG streams, random-init weights)", "config": workload(args, args.gpus),
            "impl": "reference",
            "latency_ms": {"cpu_tick": lat([x * 1e3 for x in t]), "slo": SLO_MS},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "port",
                             "sample": (f"every step = one full {P}-bed tick" if beds == P else
                                        f"every step = {beds} of the {P} beds (time budget {args.ref_budget_s:.0f} s)")
                                       + f" x {sel.popcount} members, CPU oracle port oracle/cpu_path.cpu_tick "
                                         "(PyTorch fp32; the reference has no CNN)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ B200 arm
def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2008_04063_b200.engine import EnsembleEngine, TickResult
    from paper_2008_04063_b200.parallel import MemberShardedEngine

    rank, world, local = rank_env()
    torch.cuda.set_device(local)
    member = args.mode == "member"
    if world > 1 or member:
        if world == 1:
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", str(free_port()))
            os.environ.setdefault("RANK", "0")
            os.environ.setdefault("WORLD_SIZE", "1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ranks = Ranks(world, device="cuda")

    P, hop, K, Wu = args.patients, args.hop, args.steps, args.warmup
    zoo, sel = selection(args)
    nt = Wu + K
    # this rank's beds: disjoint shards (patient mode) or all beds (member mode)
    pids = list(range(rank * P, (rank + 1) * P)) if not member else list(range(P))
    streams = streams_for(pids, hop, nt, seed=0)
    if member:
        meng = MemberShardedEngine(zoo, sel, P, rank, world, device=local, seed=0, hop=hop)
        eng = meng.engine
    else:
        meng = None
        eng = EnsembleEngine(zoo, sel, P, hop=hop, device=local, seed=0)
    eng.ingest(streams[:, :, :W - hop])
    hop_blocks = np.ascontiguousarray(streams[:, :, W - hop:].reshape(P, 3, nt, hop).transpose(2, 0, 1, 3))
    dev_blocks = torch.from_numpy(hop_blocks).cuda()
    stream = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    M_local = eng.selector.popcount

    def one_tick(i):
        eng.stage_device(dev_blocks[i].data_ptr(), stream.cuda_stream)
        eng.tick_device(stream.cuda_stream)
        if member:
            meng.reduce_device(stream)

    # ---- device-resident timing (value, tick latency)
    with torch.cuda.stream(stream):
        for i in range(Wu):
            one_tick(i)
    torch.cuda.synchronize()
    ranks.barrier()
    clocks = Clocks(local) if not args.profile_only else None
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    red_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for i in range(K):
            flush.zero_()
            evs[i][0].record(stream)
            eng.stage_device(dev_blocks[Wu + i].data_ptr(), stream.cuda_stream)
            eng.tick_device(stream.cuda_stream)
            if member:
                red_evs[i][0].record(stream)
                meng.reduce_device(stream)
                red_evs[i][1].record(stream)
            evs[i][1].record(stream)
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = ranks.max(float(sum(step_ms)))
    dev_lat = {k: ranks.max(v) for k, v in lat(step_ms).items()}
    reduce_ms = lat([a.elapsed_time(b) for a, b in red_evs]) if member else None
    ranks.barrier()
    units_per_tick = world * P if not member else P
    value = units_per_tick * K / (total_ms / 1e3)

    # ---- parity: the last timed tick's outputs vs the CPU oracle on sampled beds (rank 0)
    parity = None
    if not args.profile_only and args.parity_beds > 0:
        end = W - hop + nt * hop
        if member:
            prob_t, logit_t = meng.finished_outputs()
            if rank == 0:
                ml_all = None
                parity = parity_check_member(zoo, sel, streams, end, sample_beds(P, args.parity_beds),
                                             prob_t, logit_t)
        elif rank == 0:
            ml, prob, mlog = device_outputs(eng, P, M_local)
            parity = parity_check(zoo, sel, streams, end, sample_beds(P, args.parity_beds), ml, prob, mlog)
        ml_all = None  # noqa: F841

    # ---- per-kernel profile of one tick (events after every launch, same stream)
    reps = 5
    prof = [eng.profile_tick(stream.cuda_stream) for _ in range(reps)]
    kinds = prof[0][0]
    ms = np.mean([p[1] for p in prof], axis=0)
    flops = prof[0][2]
    conv = (kinds == 2) | (kinds == 5) | (kinds == 6)
    conv_ms, conv_flops = float(ms[conv].sum()), float(flops[conv].sum())
    pp = kinds == 5  # K4b, the polyphase conv, one launch per layer (per-layer tick)
    pp_ms, pp_flops, pp_n = float(ms[pp].sum()), float(flops[pp].sum()), int(pp.sum())
    ch = kinds == 6  # K4c, every K4b layer of the tick in one persistent launch (the c2 tick's default)
    ch_ms, ch_flops, ch_n = float(ms[ch].sum()), float(flops[ch].sum()), int(ch.sum())
    tc = kinds == 2
    tc_ms, tc_flops = float(ms[tc].sum()), float(flops[tc].sum())
    tick_ms_eager = float(ms.sum())
    cands = [(ch_ms, ch_flops, ch_n, "hb::chain_pp_kernel (K4c)", 6), (pp_ms, pp_flops, pp_n, "hb::conv_pp_kernel (K4b)", 5),
             (tc_ms, tc_flops, int(tc.sum()), "hb::conv_tc_kernel (K4)", 2)]
    dom_ms, dom_flops, dom_n, dom_name, dom_kind = max(cands, key=lambda c: c[0])
    achieved = dom_flops / (dom_ms / 1e3) / 1e12 if dom_ms > 0 else 0.0
    peak_tf, peak_sus, peak_hbm, peak_src = peaks()
    abytes = prof[0][3]
    dom_roof_ms = float(sum(max(flops[i] / (peak_tf * 1e12), abytes[i] / (peak_hbm * 1e9)) * 1e3
                            for i in range(len(kinds)) if kinds[i] == dom_kind))
    dom_hbm_bound = int(sum(1 for i in range(len(kinds))
                            if kinds[i] == dom_kind and abytes[i] / (peak_hbm * 1e9) > flops[i] / (peak_tf * 1e12)))
    traffic, ncu_meta = ncu_traffic()
    n_launch = int(len(kinds)) + (1 if member and rank == 0 else 0)

    # ---- end-to-end through the public API with pinned host buffers
    host_in = torch.empty((nt, P, 3, hop), dtype=torch.float32, pin_memory=True)
    host_in.numpy()[:] = hop_blocks
    hin = host_in.numpy()
    e2e = {}
    if not member:
        out = TickResult(eng.member_ids, torch.empty((P, M_local), pin_memory=True).numpy(),
                         torch.empty(P, pin_memory=True).numpy(), torch.empty(P, pin_memory=True).numpy())
        for i in range(Wu):
            eng.tick(hin[i], out=out)
        # (1) pipelined: tick t+1 is submitted (H2D + tick + D2H enqueued) before tick t's
        #     outputs are collected; every step's H2D and D2H stay inside the timed region
        ranks.barrier()
        t0 = time.perf_counter()
        slot = eng.submit(hin[Wu])
        for i in range(K):
            nxt = eng.submit(hin[Wu + i + 1]) if i + 1 < K else None
            eng.collect(slot, out=out)
            slot = nxt
        e2e_s = ranks.max(time.perf_counter() - t0)
        # (2) one blocking EnsembleEngine.tick per step, each host-timed: per-tick e2e latency
        ranks.barrier()
        t0 = time.perf_counter()
        step_e2e = []
        for i in range(K):
            a = time.perf_counter()
            eng.tick(hin[Wu + i], out=out)
            step_e2e.append((time.perf_counter() - a) * 1e3)
        e2e_sync_s = ranks.max(time.perf_counter() - t0)
        e2e_lat = {k: ranks.max(v) for k, v in lat(step_e2e).items()}
        e2e = {"value": units_per_tick * K / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": P * 3 * hop * 4, "d2h_bytes_per_step": P * M_local * 4 + 2 * P * 4,
               "api": "EnsembleEngine.submit/collect (tick t+1 submitted before tick t is collected)",
               "blocking_tick": {"value": units_per_tick * K / e2e_sync_s,
                                 "api": "EnsembleEngine.tick, one blocking call per step",
                                 "tick_ms": e2e_lat}}
    else:
        for i in range(Wu):
            meng.tick(hin[i])
        ranks.barrier()
        t0 = time.perf_counter()
        step_e2e = []
        for i in range(K):
            a = time.perf_counter()
            meng.tick(hin[Wu + i])
            step_e2e.append((time.perf_counter() - a) * 1e3)
        e2e_s = ranks.max(time.perf_counter() - t0)
        e2e_lat = {k: ranks.max(v) for k, v in lat(step_e2e).items()}
        e2e = {"value": units_per_tick * K / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": P * 3 * hop * 4, "d2h_bytes_per_step": 2 * P * 4 if rank == 0 else 0,
               "api": "MemberShardedEngine.tick (pinned H2D of all beds' hop, this rank's members, "
                      "NCCL reduce to rank 0, finalize, D2H of the scores on rank 0)",
               "tick_ms": e2e_lat}
    ck = clocks.stop() if clocks else None

    cpu = None
    if rank == 0 and world == 1 and not member and not args.no_cpu_baseline and not args.profile_only:
        cpu = cpu_baseline(zoo, sel, P, hop)
    extras = {}
    if rank == 0 and world == 1 and not member and not args.profile_only and not args.no_extras \
            and args.members == "c2":
        eng.close()
        extras["beds_1024"] = tick_at(zoo, sel, 1024, hop, local, K=200, e2e_ticks=100)
        from paper_2008_04063_b200.zoo import Selector
        extras["c3_full_zoo_100_beds"] = tick_at(zoo, Selector.ones(60), 100, hop, local, K=50, warm=3,
                                                 e2e_ticks=20)
        # BASELINE c1: one member (ecg-i-w32-d8, as tests/test_parity_timed_gpu.py::test_c1) for one bed
        extras["c1_one_member_one_bed"] = tick_at(zoo, Selector.from_indices(60, [10]), 1, hop, local, K=200,
                                                  e2e_ticks=100)
        extras["profiler_sweep"] = sweep_bench(local)

    roof = tick_roofline(zoo, eng.selector, P, peak_tf, peak_hbm)
    roof["frac_of_measured_p50"] = roof["ms"] / dev_lat["p50"]
    detail = {
        "tick_breakdown_ms_eager": {
            "ingest_window": float(ms[kinds == 0].sum()), "stem": float(ms[kinds == 1].sum()),
            "conv_tcgen05": conv_ms, "conv_k4c_chain": ch_ms, "conv_k4b": pp_ms, "conv_k4": tc_ms,
            "aggregate": float(ms[kinds == 3].sum() + ms[kinds == 4].sum()), "total": tick_ms_eager},
        "tick_path": ("K4c chain: window, stems (one launch), ONE persistent conv launch with the ensemble aggregation fused in"
                      if ch_n else "per-layer: one K4/K4b launch per conv layer, member lanes in graph branches"),
        "tick_launches": [int(x) for x in kinds],
        "tick_flops": float(flops.sum()),
        "tick_roofline": roof,
    }
    if member:
        detail["member_bins"] = meng.bins
        detail["nccl_reduce_ms"] = reduce_ms
        detail["nccl_reduce_bytes"] = 2 * P * 4
    detail.update(extras)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": Wu,
        "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "strong" if member else "weak",
        "vs_baseline": None, "dtype": "f16", "data": "synthetic (seeded ECG streams, random-init weights)",
        "config": workload(args, world),
        "latency_ms": {"device_tick": dev_lat, "e2e_tick": e2e.get("blocking_tick", e2e).get("tick_ms"),
                       "slo": SLO_MS, "def": "nearest-rank percentiles (runtime.py:246) over the K timed steps, "
                                             "max over ranks"},
        "per_rank_value": value / world,
        "parity": parity,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": achieved / peak_tf, "traffic": traffic, "kernel": dom_name,
                     "peak_kind": "burst (bf16_tflops; the kernel is timed in one eager tick)",
                     "frac_of_sustained": achieved / peak_sus, "peak_sustained": peak_sus,
                     "launches_per_tick": dom_n, "share_of_tick": dom_ms / tick_ms_eager, "peak_source": peak_src,
                     "time_roofline": {"frac": dom_roof_ms / dom_ms if dom_ms > 0 else None,
                                       "roofline_ms": dom_roof_ms, "measured_ms": dom_ms,
                                       "hbm_bound_launches": dom_hbm_bound,
                                       "def": "sum over the kernel's launches of max(FLOPs/burst tensor peak, "
                                              "activation bytes/HBM peak) / their measured eager ms"},
                     "achieved_def": "sum of the kernel's algorithmic FLOPs / sum of its launch ms over one tick "
                                     "(2*Cin*Cout*16*Lout*P per layer; the zero taps K4b/K4c also issue are not counted)",
                     "all_conv": {"kernels": "K4c + K4b + K4 (hb::conv_tc_kernel)",
                                  "tflops": conv_flops / (conv_ms / 1e3) / 1e12 if conv_ms > 0 else None,
                                  "share_of_tick": conv_ms / tick_ms_eager,
                                  "k4_tflops": tc_flops / (tc_ms / 1e3) / 1e12 if tc_ms > 0 else None},
                     "ncu": ncu_meta},
        "e2e": e2e,
        "gpu_launches": n_launch * K,
        "clocks": ck,
        "cpu_baseline": cpu,
        "detail": detail,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if meng is not None:
        meng.close()
    elif not extras:
        eng.close()
    if dist.is_initialized():
        dist.destroy_process_group()


def parity_check_member(zoo, sel, streams, end, beds, prob, logit) -> dict:
    """Member mode: rank 0's combined ensemble outputs (all members over all ranks) vs the oracle."""
    from oracle import cpu_path
    _, oprob, omean = cpu_path.cpu_tick(zoo, sel, streams, end, beds=beds)
    dp = float(np.abs(prob[beds] - oprob).max())
    dm = float(np.abs(logit[beds] - omean).max())
    return {"beds": len(beds), "bed_ids": beds, "max_dprob": dp, "max_dmean_logit": dm,
            "tol": {"prob": 1e-3, "logit": 2e-2}, "ok": bool(dp <= 1e-3 and dm <= 2e-2),
            "oracle": "oracle/cpu_path.cpu_tick (PyTorch fp32 CPU)"}


def main(argv=None):
    args = parse(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-execute under torch.distributed.run (rank 0 prints the line)
        cmd = launch_argv(sys.argv[1:] if argv is None else argv, args.gpus, free_port())
        sys.stdout.flush()
        os.execv(sys.executable, cmd)
    visible = None
    if args.impl == "b200":
        import torch
        visible = torch.cuda.device_count()
    why = check_world(args, visible=visible)
    if why:
        print(f"bench.py: refusing to run: {why}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
