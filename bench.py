#!/usr/bin/env python
"""Benchmark of the HOLMES serving hot path on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1], "c2"): a 4-member ResNet1D ensemble
(ecg-i-w32-d8, ecg-i-w64-d4, ecg-ii-w32-d8, ecg-iii-w32-d8 of the paper's
60-member zoo) serving 64 beds x 3 ECG leads at 250 Hz; every 1 s tick each
bed's latest 7500-sample window is z-normalised and scored by every member and
the member sigmoids are averaged.  One *step* = one tick over all beds.
Synthetic streams (seeded), random-init synthetic weights (no checkpoints).

  value  : patient-windows/s over all ranks, inputs already in HBM, device
           time (CUDA events per step, L2 flushed by a 256 MiB write between
           steps), max over ranks.
  e2e    : same metric through the public API with pinned host buffers (H2D
           of each tick's samples + D2H of its scores inside the timed region),
           host wall clock, max over ranks: `EnsembleEngine.submit/collect`
           (tick t+1 enqueued before tick t is collected), and under
           `blocking_tick` one blocking `EnsembleEngine.tick` per step.
  roofline: the polyphase tcgen05 conv kernel K4b (the dominant kernel; the
           wide layers and heads run on K4, reported under all_conv) —
           algorithmic conv FLOPs / event-timed launch duration, launched eagerly with an event
           after every kernel on the serving stream right after the timed
           region; peak = MEASURED_PEAKS.json sustained dense 16-bit TFLOP/s.
  cpu_baseline: the CPU oracle port of the same tick (PyTorch fp32, all host
           threads) on a bounded patient sample, rank 0 at N=1.

Multi-GPU: patient-sharded (each rank serves its own 64 beds; no collective on
the data path — the reference's units are independent), "scaling": "weak".
`--impl reference` times the CPU oracle port on the host cores (the reference
has no CNN and no GPU path; its own scorer is an analytic stand-in).
"""
from __future__ import annotations

import argparse
import json
import os
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)  # >= 1000 ticks per config
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--patients", type=int, default=64, help="beds per GPU")
    ap.add_argument("--hop", type=int, default=250)
    ap.add_argument("--cpu-patients", type=int, default=8, help="CPU baseline sample size")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile-only", action="store_true", help="short run for ncu (no clocks / cpu)")
    ap.add_argument("--no-extras", action="store_true", help="skip the 1024-bed and profiler-sweep side measurements")
    return ap.parse_args()


def workload(args):
    return {
        "workload": "c2: 4-member ResNet1D ensemble, 64-bed 250 Hz 3-lead ECG, 7500-sample sliding window, 1 s tick",
        "members": ["ecg-i-w32-d8", "ecg-i-w64-d4", "ecg-ii-w32-d8", "ecg-iii-w32-d8"],
        "patients_per_gpu": args.patients,
        "window": 7500,
        "hop": args.hop,
        "aggregation": "mean of member sigmoids (+ mean latent)",
        "precision": "fp16 operands, fp32 accumulate; fp16 activations",
        "l2": "flushed between timed steps (256 MiB device write)",
        "parallelism": f"patient-sharded x{args.gpus}",
    }


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
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            d = json.load(fh)
        return float(d["bf16_tflops_sustained"]), float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json, sustained)"
    except (OSError, KeyError, ValueError):
        return 1400.0, 6650.0, "fallback (B200_PROFILING.md)"


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


def cpu_baseline(zoo, sel, n_patients, seed=0):
    import torch
    from oracle.cpu_path import cpu_tick, params_for
    from paper_2008_04063_b200 import synth
    torch.set_num_threads(os.cpu_count() or 1)
    for i in sel.indices():
        params_for(zoo.profiles[i], seed)
    streams = synth.ecg_block(seed, n_patients, 3, 0, 7500)
    cpu_tick(zoo, sel, streams[:1], 7500, seed=seed)  # warm
    t0 = time.perf_counter()
    cpu_tick(zoo, sel, streams, 7500, seed=seed)
    dt = time.perf_counter() - t0
    return {"value": n_patients / dt, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "port",
            "sample": f"{n_patients} patient-windows x 4 members (one c2 tick subset), PyTorch fp32 CPU oracle, "
                      f"{dt:.2f} s"}


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
            "def": "sum_layers max(FLOPs/sustained tensor peak, (in+out+shortcut) fp16 bytes/HBM peak)"}


def tick_at(zoo, sel, P, hop, device, K=30, warm=5):
    """North-star side measurement: the same ensemble at P beds (graph tick, device time, L2 flushed)."""
    import torch
    from paper_2008_04063_b200.engine import EnsembleEngine
    eng = EnsembleEngine(zoo, sel, P, hop=hop, device=device)
    eng.ingest((np.random.default_rng(1).standard_normal((P, 3, 7500)) * 0.3).astype(np.float32))
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
    # the memory-bound stream kernels at this scale: achieved HBM GB/s of ingest+window
    # (algorithmic bytes: append 8 B + window 4 B read + 2 B write per sample) and aggregate
    kinds, kms, _, kbytes = eng.profile_tick(st.cuda_stream)
    torch.cuda.synchronize()
    stream_k = {}
    for kind, name in ((0, "ingest_window"), (3, "aggregate")):
        sel_k = kinds == kind
        if sel_k.any():
            tms = float(kms[sel_k].sum())
            stream_k[name] = {"ms": tms, "bytes": float(kbytes[sel_k].sum()),
                              "gbs": float(kbytes[sel_k].sum()) / (tms / 1e3) / 1e9 if tms > 0 else None}
    eng.close()
    return {"patients": P, "tick_ms_p50": pct(t, 50), "tick_ms_p99": pct(t, 99),
            "patient_windows_per_s": P / (float(np.mean(t)) / 1e3),
            "tflops": flops / (float(np.mean(t)) / 1e3) / 1e12, "ticks": K, "stream_kernels_eager": stream_k}


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
    # CPU oracle (same algorithm, numpy, 1 core) on a bounded sample of the n=10 sweep
    z = generate_zoo(1, [8, 16, 32, 64, 128], [2, 4], seed=3)
    coh = hc.synthesize_cohort(z, 10000, 10000, 0.5, 0)
    vals = np.arange(1, 65)
    t0 = time.perf_counter()
    oauc.sweep(coh.labels, coh.scores, vals)
    dt = time.perf_counter() - t0
    out["cpu_oracle"] = {"candidates_per_s": len(vals) / dt, "cores": 1, "sample": "64 candidates of n=10, N=20000"}
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch
    from oracle.cpu_path import cpu_tick, params_for
    from paper_2008_04063_b200 import synth
    from paper_2008_04063_b200.zoo import Selector, holmes_zoo
    torch.set_num_threads(os.cpu_count() or 1)
    zoo, sel = holmes_zoo(), Selector.from_indices(60, MEMBERS)
    for i in sel.indices():
        params_for(zoo.profiles[i])
    n = max(1, args.cpu_patients // 2)
    streams = synth.ecg_block(0, n, 3, 0, 7500 + args.hop * (args.steps + args.warmup))
    end = 7500
    for _ in range(args.warmup):
        cpu_tick(zoo, sel, streams, end)
        end += args.hop
    t0 = time.perf_counter()
    for _ in range(args.steps):
        cpu_tick(zoo, sel, streams, end)
        end += args.hop
    dt = time.perf_counter() - t0
    value = n * args.steps / dt
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": workload(args), "impl": "reference",
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": torch.get_num_threads(), "kind": "port",
                             "sample": f"{n} patients per step (bounded sample of the 64-bed tick), "
                                       "CPU oracle port (the reference has no CNN)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_b200(args):
    import torch
    import torch.distributed as dist
    from paper_2008_04063_b200 import synth
    from paper_2008_04063_b200.engine import EnsembleEngine, TickResult
    from paper_2008_04063_b200.zoo import Selector, holmes_zoo

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if world > 1:
            dist.barrier()

    def allmax(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    P, hop, K, Wu = args.patients, args.hop, args.steps, args.warmup
    zoo, sel = holmes_zoo(), Selector.from_indices(60, MEMBERS)
    eng = EnsembleEngine(zoo, sel, P, hop=hop, device=local, seed=0)
    # synthetic streams for this rank's beds (patient ids offset by rank: shards are disjoint)
    pids = list(range(rank * P, (rank + 1) * P))
    nt = Wu + K
    prefill = synth.ecg_block(0, pids, 3, 0, 7500)
    eng.ingest(prefill)
    rng = np.random.default_rng(rank)
    hop_blocks = (rng.standard_normal((nt, P, 3, hop)) * 0.3).astype(np.float32)  # tick payloads
    dev_blocks = torch.from_numpy(hop_blocks).cuda()
    stream = torch.cuda.Stream()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    # ---- device-resident timing (value, tick latency)
    with torch.cuda.stream(stream):
        for i in range(Wu):
            eng.stage_device(dev_blocks[i].data_ptr(), stream.cuda_stream)
            eng.tick_device(stream.cuda_stream)
    torch.cuda.synchronize()
    barrier()
    clocks = Clocks(local) if not args.profile_only else None
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    torch.cuda.synchronize()
    with torch.cuda.stream(stream):
        for i in range(K):
            flush.zero_()
            evs[i][0].record(stream)
            eng.stage_device(dev_blocks[Wu + i].data_ptr(), stream.cuda_stream)
            eng.tick_device(stream.cuda_stream)
            evs[i][1].record(stream)
    torch.cuda.synchronize()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = allmax(float(sum(step_ms)))
    barrier()
    p50, p95, p99 = (allmax(pct(step_ms, q)) for q in (50, 95, 99))
    value = world * P * K / (total_ms / 1e3)

    # ---- per-kernel profile of the same tick (events after every launch, same stream)
    reps = 5
    prof = [eng.profile_tick(stream.cuda_stream) for _ in range(reps)]
    kinds = prof[0][0]
    ms = np.mean([p[1] for p in prof], axis=0)
    flops = prof[0][2]
    conv = (kinds == 2) | (kinds == 5)
    conv_ms, conv_flops = float(ms[conv].sum()), float(flops[conv].sum())
    pp = kinds == 5  # K4b, the polyphase conv: the dominant kernel of the tick
    pp_ms, pp_flops, pp_n = float(ms[pp].sum()), float(flops[pp].sum()), int(pp.sum())
    tc = kinds == 2
    tc_ms, tc_flops = float(ms[tc].sum()), float(flops[tc].sum())
    tick_ms_eager = float(ms.sum())
    achieved = pp_flops / (pp_ms / 1e3) / 1e12 if pp_ms > 0 else conv_flops / (conv_ms / 1e3) / 1e12
    peak_tf, peak_hbm, peak_src = peaks()
    # K4b against its own per-launch roofline: sum over its launches of
    # max(FLOPs / tensor peak, algorithmic activation bytes / HBM peak), over the measured time
    abytes = prof[0][3]
    pp_roof_ms = float(sum(max(flops[i] / (peak_tf * 1e12), abytes[i] / (peak_hbm * 1e9)) * 1e3
                           for i in range(len(kinds)) if kinds[i] == 5))
    pp_hbm_bound = int(sum(1 for i in range(len(kinds))
                           if kinds[i] == 5 and abytes[i] / (peak_hbm * 1e9) > flops[i] / (peak_tf * 1e12)))
    traffic, ncu_meta = ncu_traffic()
    n_launch = int(len(kinds))

    # ---- end-to-end through the public API with pinned host buffers
    M = sel.popcount
    host_in = torch.empty((nt, P, 3, hop), dtype=torch.float32, pin_memory=True)
    host_in.numpy()[:] = hop_blocks
    out = TickResult(eng.member_ids, torch.empty((P, M), pin_memory=True).numpy(),
                     torch.empty(P, pin_memory=True).numpy(), torch.empty(P, pin_memory=True).numpy())
    hin = host_in.numpy()
    for i in range(Wu):
        eng.tick(hin[i], out=out)
    # (1) pipelined: tick t+1 is submitted (H2D + tick + D2H enqueued) before tick t's
    #     outputs are collected; every step's H2D and D2H stay inside the timed region
    barrier()
    t0 = time.perf_counter()
    slot = eng.submit(hin[Wu])
    for i in range(K):
        nxt = eng.submit(hin[Wu + i + 1]) if i + 1 < K else None
        eng.collect(slot, out=out)
        slot = nxt
    e2e_s = allmax(time.perf_counter() - t0)
    # (2) one blocking EnsembleEngine.tick per step (the real-time serving call)
    for i in range(Wu):
        eng.tick(hin[i], out=out)
    barrier()
    t0 = time.perf_counter()
    for i in range(K):
        eng.tick(hin[Wu + i], out=out)
    e2e_sync_s = allmax(time.perf_counter() - t0)
    ck = clocks.stop() if clocks else None
    e2e_value = world * P * K / e2e_s
    e2e_sync_value = world * P * K / e2e_sync_s
    h2d = P * 3 * hop * 4
    d2h = P * M * 4 + 2 * P * 4

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and not args.profile_only:
        cpu = cpu_baseline(zoo, sel, args.cpu_patients)
    extras = {}
    if rank == 0 and world == 1 and not args.profile_only and not args.no_extras:
        eng.close()
        extras["beds_1024"] = tick_at(zoo, sel, 1024, hop, local, K=200)
        extras["c3_full_zoo_100_beds"] = tick_at(zoo, Selector.ones(60), 100, hop, local, K=50, warm=3)
        extras["profiler_sweep"] = sweep_bench(local)

    cfg = workload(args)
    cfg["tick_latency_ms"] = {"p50": p50, "p95": p95, "p99": p99, "slo": SLO_MS}
    cfg["tick_breakdown_ms_eager"] = {
        "ingest_window": float(ms[kinds == 0].sum()), "stem": float(ms[kinds == 1].sum()),
        "conv_tcgen05": conv_ms, "conv_k4b": pp_ms, "conv_k4": tc_ms,
        "aggregate": float(ms[kinds == 3].sum() + ms[kinds == 4].sum()),
        "total": tick_ms_eager}
    cfg["tick_flops"] = float(flops.sum())
    roof = tick_roofline(zoo, sel, P, peak_tf, peak_hbm)
    roof["frac_of_measured_p50"] = roof["ms"] / p50
    cfg["tick_roofline"] = roof
    cfg.update(extras)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": Wu,
        "ms_per_step": total_ms / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f16", "data": "synthetic (seeded ECG streams, random-init weights)", "config": cfg,
        "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak_tf, "unit": "TFLOP/s",
                     "frac": achieved / peak_tf, "traffic": traffic, "kernel": "hb::conv_pp_kernel (K4b)",
                     "launches_per_tick": pp_n, "share_of_tick": pp_ms / tick_ms_eager, "peak_source": peak_src,
                     "time_roofline": {"frac": pp_roof_ms / pp_ms if pp_ms > 0 else None, "roofline_ms": pp_roof_ms,
                                       "measured_ms": pp_ms, "hbm_bound_launches": pp_hbm_bound,
                                       "def": "sum over K4b launches of max(FLOPs/tensor peak, activation bytes/HBM peak) "
                                              "/ their measured eager ms"},
                     "achieved_def": "sum K4b algorithmic FLOPs / sum K4b launch ms over one tick "
                                     "(2*Cin*Cout*16*Lout*P per layer; the zero taps K4b also issues are not counted)",
                     "all_conv": {"kernels": "K4b + K4 (hb::conv_tc_kernel)", "tflops": conv_flops / (conv_ms / 1e3) / 1e12,
                                  "frac": conv_flops / (conv_ms / 1e3) / 1e12 / peak_tf,
                                  "share_of_tick": conv_ms / tick_ms_eager,
                                  "k4_tflops": tc_flops / (tc_ms / 1e3) / 1e12 if tc_ms > 0 else None},
                     "ncu": ncu_meta},
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "EnsembleEngine.submit/collect (tick t+1 submitted before tick t is collected)",
                "blocking_tick": {"value": e2e_sync_value, "api": "EnsembleEngine.tick, one blocking call per step"}},
        "gpu_launches": n_launch * K,
        "clocks": ck,
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if not extras:
        eng.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
