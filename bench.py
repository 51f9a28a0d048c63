#!/usr/bin/env python
"""Benchmark of the batched unsteady-DSMC step on B200 (BASELINE.json metric:
particle-steps/s per B200, all runs batched; % of HBM roofline).

One "step" = one pass of the whole hot path (inflow Generation, Motion,
Enumeration, Indexing/LCR, NTC Interaction, Sampling, reorder) over all
n runs of the batch.  Default workload: configs[3] (c4, 3D equilibrium box
64^3 x 10 ppc) at n = 256 runs, the largest batched configuration (671M
particles); see DESIGN.md "Measurement" for why c4 is the headline.

Multi-GPU (torchrun): runs are independent (PSIR), so each
rank takes n runs with run ids offset by rank*n -- weak scaling, no
collective on the data path; time = max over ranks.

--impl reference times the CPU oracle (test infrastructure, oracle/) on a
bounded sample of the same workload on this host's cores.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import configs  # noqa: E402

PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
# arithmetic types of the path (R6): fp32 particle state and majorant,
# fp64 candidate count, acceptance test and sampled sums
DTYPE = "f32 (state, majorant) + f64 (NTC count, acceptance, sums)"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} logical CPUs)"
    except OSError:
        pass
    return None


FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--n-runs", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-batches", type=int, default=0,
                    help="sub-batches (contexts) the e2e leg streams the runs in (0: n/16 when n >= 64, else 1)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--timed-steps", type=int, default=4, help="steps of the per-kernel event-timed pass")
    ap.add_argument("--reorder-every", type=int, default=None, help="physical reorder period K (problem parameter)")
    return ap.parse_args()


def workload(args, rank=0):
    kw = {}
    if args.config == "c4":
        kw = dict(n_runs=args.n_runs or 256, n_steps=100)
    elif args.n_runs:
        kw = dict(n_runs=args.n_runs)
    p = configs.get(args.config, **kw)
    p["run_id0"] = rank * p["n_runs"]
    if args.reorder_every is not None:
        p["reorder_every"] = args.reorder_every
    return p


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback"


class Clocks:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    def __init__(self, index=0):
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_{os.getpid()}.csv")
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}",
                 "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        self.f.close()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def algorithmic_bytes(p, kernel, live, cells, accepted, sample, reorder):
    """Bytes a kernel must move per launch.
    live: live particles of the batch, cells: n*Nc, accepted: pairs this step."""
    D = p["dim"]
    if kernel == "k_motion":      # R pos(4D)+vel(12), W pos(4D), W key(4); counts 4/cell
        return live * (8 * D + 16) + 4 * cells
    if kernel == "k_scatter":     # R key 4, W LCR 4; cursor R+W 8/cell
        return live * 8 + 8 * cells
    if kernel == "k_collide":     # R ends 4 + gmax 4 /cell, R LCR 4 + vel 12, W vel of collided
        b = live * 16 + 8 * cells + 2 * accepted * 12
        if sample:
            b += 40 * cells
        if reorder:               # R pos, W pos + vel to the other half
            b += live * (4 * D + 4 * D + 12)
        return b
    if kernel == "k_scan_reduce":
        return 4 * cells
    if kernel == "k_scan_down":
        return 8 * cells
    if kernel == "k_zero":
        return 4 * cells
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_cs_9902024_b200 import dsmc

    from paper_cs_9902024_b200 import runs
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")
    p = runs.shard(workload(args, 0), rank, world)   # weak scaling: n runs per GPU, ids offset
    sim = dsmc.Simulation(p, device=f"cuda:{local}")
    sim.generate()
    stream = sim.stream
    K, W = args.steps, args.warmup
    sim.step(W)
    torch.cuda.synchronize()
    _, st0 = sim.status()
    clocks = Clocks(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    sim.step(K)
    e1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    _, st1 = sim.status()
    psteps = sum(b["particle_steps"] - a["particle_steps"] for a, b in zip(st0, st1))
    accepted = sum(b["accepted"] - a["accepted"] for a, b in zip(st0, st1)) / K
    cands = sum(b["candidates"] - a["candidates"] for a, b in zip(st0, st1)) / K
    live_avg = psteps / K
    ms_max = runs.max_over_ranks(ms)
    psteps_all = runs.sum_over_ranks(float(psteps))
    value = psteps_all / (ms_max / 1e3)
    kps = sim.kernels_per_step()

    # per-kernel CUDA-event timing pass (same work, kernel by kernel) for the roofline
    timed = sim.step_timed(args.timed_steps)
    _, st2 = sim.status()
    steps_done = st2[0]["step"]
    cells = sim.R * sim.Nc
    # fraction of timed steps that sample / reorder
    S, Kr = configs.sample_every(p), p["reorder_every"] or 10 ** 9
    first = steps_done - args.timed_steps
    n_sample = sum(1 for s in range(first, steps_done) if (s + 1) % S == 0)
    n_reorder = sum(1 for s in range(first, steps_done) if (s + 1) % Kr == 0)
    hbm, peak_kind = peaks()
    kern = {}
    for name, (tms, cnt) in timed.items():
        avg = tms / cnt
        b = (algorithmic_bytes(p, name, live_avg, cells, accepted, False, False) * (cnt - n_sample - n_reorder)
             + algorithmic_bytes(p, name, live_avg, cells, accepted, True, False) * n_sample
             + algorithmic_bytes(p, name, live_avg, cells, accepted, False, True) * n_reorder) / cnt \
            if name == "k_collide" else algorithmic_bytes(p, name, live_avg, cells, accepted, False, False)
        kern[name] = dict(ms=avg, gbs=(b / (avg / 1e3) / 1e9) if b else None, bytes=b)
    step_ms_sum = sum(v["ms"] for v in kern.values())
    # Interaction runs as two launches (warp tiles, then the heavy tiles they hand
    # over); the roofline treats them as one kernel with k_collide's byte count
    # (sparse problems add the triage that lists the tiles with work)
    parts = [k for k in ("k_collide_triage", "k_collide", "k_collide_heavy") if k in kern]
    cand = {k: v for k, v in kern.items() if k not in parts}
    if "k_collide" in kern:
        ms = sum(kern[k]["ms"] for k in parts)
        b = kern["k_collide"]["bytes"]
        name = "+".join(parts)
        cand[name] = dict(ms=ms, gbs=b / (ms / 1e3) / 1e9 if b else None, bytes=b)
    dom = max(cand, key=lambda k: cand[k]["ms"])
    d = cand[dom]
    roof = {"bound": "hbm", "kernel": dom, "achieved": round(d["gbs"], 1) if d["gbs"] else None,
            "peak": hbm, "peak_kind": peak_kind, "unit": "GB/s",
            "frac": round(d["gbs"] / hbm, 4) if d["gbs"] else None, "traffic": None,
            "share_of_step": round(d["ms"] / step_ms_sum, 3),
            "kernels": {k: {"ms": round(v["ms"], 4), "GB/s": round(v["gbs"], 1) if v["gbs"] else None,
                            "share": round(v["ms"] / step_ms_sum, 3)} for k, v in kern.items()}}
    # the two phases of the north-star targets, algorithmic bytes over
    # summed kernel time, against the measured copy peak and the 8 TB/s nominal
    phases = {}
    for ph, names in (("motion+sort", ("k_zero", "k_motion", "k_scan_reduce", "k_scan_partials", "k_scan_down",
                                        "k_scatter")),
                      ("collide+sample", ("k_collide_triage", "k_collide", "k_collide_heavy"))):
        ms = sum(kern[k]["ms"] for k in names if k in kern)
        b = sum(kern[k]["bytes"] or 0 for k in names if k in kern)
        if ms > 0:
            gbs = b / (ms / 1e3) / 1e9
            phases[ph] = {"ms": round(ms, 4), "GB/s": round(gbs, 1), "frac_measured": round(gbs / hbm, 4),
                          "frac_8TBs": round(gbs / 8000.0, 4)}
    roof["phases"] = phases
    traffic_path = os.path.join(ROOT, "profiles", f"traffic_{args.config}.json")
    if os.path.exists(traffic_path):
        try:
            tr = json.load(open(traffic_path))
            roof["traffic"] = sum(tr.get(k, 0.0) for k in dom.split("+")) or None
        except Exception:
            pass

    # end-to-end through the C ABI with host buffers: the batch state (positions,
    # velocities, majorants) uploaded from pinned host memory, K steps, explicit
    # Sampling, the one exchange, the ensemble macros to host.  The runs are
    # independent, so the batch is streamed in B sub-batches,
    # one context (stream, graph) each: sub-batch b+1's upload (host-synchronous on
    # its own stream) overlaps sub-batch b's steps, and the exchange gathers the B
    # blocks of slot sums in ascending run id -- bit-identical to one context
    # (tests/test_gpu_parity_r2.py::test_gathered_ensemble_equals_single_context).
    e2e = None
    if not args.no_e2e:
        # default: sub-batches of 32 runs (c4 n = 256, e2e G particle-steps/s for B = 1 / 2 / 4 / 8:
        # 20.1 / 26.0 / 29.8 / 33.2; the PCIe upload of the state is then the critical path)
        B = args.e2e_batches or (sim.R // 16 if sim.R >= 64 and sim.R % 16 == 0 else 1)
        if sim.R % B:
            B = 1
        m = sim.R // B
        host = []
        nbytes_h2d = 0
        for r in range(sim.R):
            s_ = sim.get_state(r)
            pinned = {}
            for k in ("x", "y", "z", "vx", "vy", "vz"):
                if k in ("y", "z") and "xyz".index(k) >= p["dim"]:
                    continue
                t = torch.from_numpy(s_[k]).pin_memory()
                pinned[k] = t
                nbytes_h2d += t.numel() * 4
            gm = torch.from_numpy(sim.get_gmax(r)).pin_memory()
            nbytes_h2d += gm.numel() * 4
            host.append((len(s_["x"]), pinned, gm))
        step0 = st2[0]["step"]
        subs = []
        for b in range(B):
            q = dict(p)
            q["n_runs"] = m
            q["run_id0"] = p["run_id0"] + b * m
            subs.append(dsmc.Simulation(q, device=f"cuda:{local}", stream=torch.cuda.Stream(device=f"cuda:{local}")))
        sa = [s.status()[1] for s in subs]
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for b, s in enumerate(subs):
            for j in range(m):
                n, pin, gm = host[b * m + j]
                _set_state_pinned(s, dsmc, j, n, pin, step0, gm)
            s.step(K)
        for s in subs:
            s.sample(0)
        torch.cuda.synchronize()                 # every sub-batch's stream
        # the paper's one exchange: the slot sums of every sub-batch
        # and every rank gathered in run order (NCCL all-gather), then the ensemble
        local_sums = torch.stack([s.slot_sums_device(0) for s in subs])
        g = runs.gather_slot_sums(local_sums).reshape(-1, *local_sums.shape[1:])
        macros = subs[0].read_macros_gathered(0, g, g.shape[0])
        t1 = time.perf_counter()
        sb = [s.status()[1] for s in subs]
        ps_e2e = sum(y["particle_steps"] - x["particle_steps"] for a_, b_ in zip(sa, sb) for x, y in zip(a_, b_))
        e2e_val = runs.sum_over_ranks(ps_e2e) / runs.max_over_ranks(t1 - t0)
        e2e = {"value": e2e_val, "unit": "particle-steps/s", "h2d_bytes_per_step": nbytes_h2d // K,
               "d2h_bytes_per_step": macros.nbytes // K, "sub_batches": B,
               "what": f"{B} sub-batch context(s) of {m} runs: set_state + set_gmax (pinned host) of each run, "
                       "K graph steps (sub-batch b+1's upload overlaps sub-batch b's steps), dsmc_sample, "
                       "gather of the slot sums over sub-batches and ranks, dsmc_read_macros_gathered (macros to host)"}
        del subs

    rc, _ = sim.status(raise_on_fault=False)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(p)
    if rank == 0:
        line = {
            "metric": "particle-steps/sec per B200 (all runs batched); % of HBM roofline",
            "value": value, "unit": "particle-steps/s", "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": DTYPE, "data": "synthetic",
            "config": {"workload": f"{args.config}: " + configs.PRESETS[args.config].__doc__.split("\n")[0],
                       "n_runs_per_gpu": p["n_runs"], "cells_per_run": configs.n_cells(p),
                       "particles_per_step": live_avg, "reorder_every": p["reorder_every"],
                       "sample_every": S, "l2": "inputs larger than L2 (state %.1f GB)" % (
                           sum(getattr(sim.sizes, k) for k in ("P", "key", "lcr", "cell")) / 1e9),
                       "parallelism": f"runs sharded over {world} GPU(s), no collective"},
            "collisions": {"accepted_per_step": accepted, "candidates_per_step": cands},
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": kps * K,
            "kernels_per_step": kps, "clocks": clk, "status": rc,
        }
        print(json.dumps(line))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def _set_state_pinned(sim, dsmc, r, n, pin, step, gmax=None):
    """dsmc_set_state (and dsmc_set_gmax) straight from pinned host tensors (alive = NULL)."""
    import ctypes as C
    ptr = {k: C.c_void_p(v.data_ptr()) for k, v in pin.items()}
    args = [ptr.get(k) for k in ("x", "y", "z", "vx", "vy", "vz")]
    L = dsmc.load_library()
    dsmc._check(L.dsmc_set_state(sim.h, r, n, *args, None, step))
    if gmax is not None:
        dsmc._check(L.dsmc_set_gmax(sim.h, r, C.c_void_p(gmax.data_ptr())))


def cpu_baseline(p, budget_s=12.0):
    """The oracle as it stands, single-threaded, on run 0 of the same workload
    for as many steps as fit in ~budget_s (bounded sample)."""
    from oracle import oracle
    o = oracle.OracleRun(p, p["run_id0"])
    o.fill()
    steps = 0
    t0 = time.perf_counter()
    ps = 0
    while True:
        n_before = o.n
        o.step(1)
        ps += n_before
        steps += 1
        if time.perf_counter() - t0 > budget_s or steps >= configs.n_steps(p):
            break
    el = time.perf_counter() - t0
    out = {"value": ps / el, "unit": "particle-steps/s", "cores": 1, "kind": "oracle", "cpu": cpu_model(),
           "sample": f"run {p['run_id0']} of the same workload, steps 0..{steps - 1} ({ps} particle-steps, {el:.1f} s)"}
    psir = cpu_psir(p, budget_s)
    if psir:
        psir["speedup_vs_1"] = psir["value"] / out["value"]
        q, S = psir["threads"], psir["speedup_vs_1"]
        # Eq. 4 solved for the parallel fraction alpha at the measured speedup
        psir["eq4_alpha"] = q * (1.0 - 1.0 / S) / (q - 1.0) if q > 1 else None
        out["psir"] = psir
    return out


def cpu_psir(p, budget_s=12.0):
    """the paper's first level (PSIR) on the host cores --
    one oracle run per thread (runs run_id0 .. run_id0 + q - 1, independent), every
    thread stepping its run for ~budget_s; the oracle's C calls release the GIL.
    Returns the aggregate particle-steps/s, or None on a one-core host."""
    import threading
    from oracle import oracle
    try:
        q = len(os.sched_getaffinity(0))
    except Exception:
        q = os.cpu_count() or 1
    if q < 2:
        return None
    orcs = [oracle.OracleRun(p, p["run_id0"] + t) for t in range(q)]
    done = [0] * q
    steps = [0] * q
    go = threading.Barrier(q + 1)
    t_end = [0.0]

    def work(t):
        o = orcs[t]
        o.fill()
        go.wait()
        while time.perf_counter() < t_end[0] and steps[t] < configs.n_steps(p):
            n_before = o.n
            o.step(1)
            done[t] += n_before
            steps[t] += 1

    th = [threading.Thread(target=work, args=(t,)) for t in range(q)]
    for x in th:
        x.start()
    t_end[0] = time.perf_counter() + 1e9        # until the barrier: set below
    go.wait()
    t0 = time.perf_counter()
    t_end[0] = t0 + budget_s
    for x in th:
        x.join()
    el = time.perf_counter() - t0
    return {"value": sum(done) / el, "threads": q,
            "sample": f"runs {p['run_id0']}..{p['run_id0'] + q - 1}, one per thread, {min(steps)}-{max(steps)} "
                      f"steps each ({sum(done)} particle-steps, {el:.1f} s)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    p = workload(args, 0)
    from oracle import oracle
    o = oracle.OracleRun(p, 0)
    o.fill()
    o.step(args.warmup)
    t0 = time.perf_counter()
    ps = 0
    for _ in range(args.steps):
        ps += o.n
        o.step(1)
    el = time.perf_counter() - t0
    v = ps / el
    print(json.dumps({
        "impl": "reference", "metric": "particle-steps/sec per B200 (all runs batched); % of HBM roofline",
        "value": v, "unit": "particle-steps/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": DTYPE, "data": "synthetic",
        "config": {"workload": f"{args.config} (oracle sample: run 0 of the batch)"},
        "cpu_baseline": {"value": v, "unit": "particle-steps/s", "cores": 1, "kind": "oracle", "cpu": cpu_model(),
                         "sample": f"run 0 only, steps {args.warmup}..{args.warmup + args.steps - 1}"},
        "e2e": {"value": v, "unit": "particle-steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
