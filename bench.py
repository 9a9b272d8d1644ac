#!/usr/bin/env python
"""bench.py — core-Hamiltonian assembly + spectrum on B200 (arXiv 1408.3839 hot path).

One step = one full pass of the hot path for one seeded BASELINE system: L0 scan,
lattice-summed Newton potential, GTO profiles, kinetic/overlap/nuclear Galerkin
blocks, H = 0.5 Lap - Nuc, S = Mass, then (periodic) the lattice DFT + batched
pencils or (box) the dense pencil; eigenvalues land in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c5] [--impl b200|reference]

The headline workload is c5 (BASELINE configs[4], the largest system: (16,16,16) cells,
N_b = 32768); the same line carries c3 (the most arithmetic: dense 1024 x 1024 box pencil)
and the time-vs-L rows of the metric (whole path, periodic chains L = 128 ... 32768).
N > 1 is launched by torchrun; ranks split the k-points of the periodic spectrum
(paper_1408_3839_b200/dist.py) and all-gather the eigenvalues: strong scaling of one
system. Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1408_3839_b200.system import make_config  # noqa: E402
from paper_1408_3839_b200.workmodel import roofline, stage_work  # noqa: E402

METRIC = "core-Hamiltonian assembly+spectrum time (ms) vs L; Galerkin entries/s; % roofline"
WORKLOAD_DESC = {
    "c1": "open-box (8,1,1) chain, m0=4, n=(32,256,256)/cell, R_N=25, dense 32x32 pencil",
    "c2": "periodic (32,1,1) supercell, m0=8, n=(32,256,256)/cell, R_N=29, 32 k-point 8x8 pencils",
    "c3": "open-box (128,1,1) chain, m0=8, n=(64,256,256)/cell, R_N=33, dense 1024x1024 pencil",
    "c4": "periodic (512,1,1) supercell, 4 nuclei, m0=16, n=(64,384,384)/cell, R_N=33, 512 k-point 16x16 pencils",
    "c5": "periodic (16,16,16) supercell, m0=8, n=64/cell, R_N=33, 3-level lattice DFT, 4096 k-point 8x8 pencils",
}


def load_peaks():
    peaks = {"hbm_gbs": 6650.0, "hbm_src": "fallback (B200_PROFILING.md)"}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        peaks["hbm_gbs"] = float(d["hbm_gbs"])
        peaks["hbm_src"] = "measured (MEASURED_PEAKS.json)"
    fp = os.path.join(ROOT, "profiles", "fp64_peak.json")
    if os.path.exists(fp):
        d = json.load(open(fp))
        peaks["fp64_tflops"] = float(d["dmma_tflops"])
        peaks["fp64_src"] = "measured DMMA (profiles/fp64_peak.json)"
    else:
        peaks["fp64_tflops"] = 37.0
        peaks["fp64_src"] = "nominal B200 FP64 tensor (no measurement)"
    return peaks


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax, "reasons": sorted(reasons),
                "samples": len(sm)}


def measured_traffic(workload, stage):
    """DRAM bytes per launch of `stage` from the latest committed `ncu --set full` summary
    (profiles/rNN_traffic.json, tools/summarize_profiles.py), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
    for f in reversed(files):
        d = json.load(open(f)).get(workload, {})
        if stage in d:
            return d[stage]["dram_bytes_per_launch"]
    return None


def workload_config(workload, sysobj, world):
    """The `config` object both arms print (identical keys and values for one workload)."""
    periodic = sysobj.notes["periodic"]
    return {"workload": workload, "desc": WORKLOAD_DESC[workload], "L": list(sysobj.L),
            "n_per_cell": list(sysobj.n), "m0": sysobj.m0, "R_N": sysobj.rank_N,
            "N_b": sysobj.basis_count, "k_points": sysobj.lattice_count if periodic else 0,
            "exponent_draw": sysobj.notes["exponent_draw"], "seed": sysobj.notes["seed"],
            "parallelism": (f"k-point shards x{world}" if periodic else f"replicas x{world}"),
            "l2": "GPU arm: flushed between timed iterations (256 MB write); CPU arm: n/a"}


def pick_cpu_impl(sysobj):
    """Oracle-X built on this host with the reference's flags (-O3 -march=native, BASELINE.md;
    bit-identical to the reference's own code on isotropic grids, tests/test_oracle_pinning.py),
    else the prebuilt x86-64-v3 Oracle-R (isotropic) / Oracle-X."""
    from oracle.binding import native_oracle, oracle, reference
    nat = native_oracle()
    if nat is not None:
        return nat, "port", "Oracle-X, -O3 -march=native built on this host"
    iso = len(set(sysobj.n)) == 1 and len(set(sysobj.nbar)) == 1
    ref = reference() if iso else None
    if ref is not None:
        return ref, "reference", "Oracle-R (reference sources), prebuilt -O3 -march=x86-64-v3"
    return oracle(), "port", "Oracle-X, prebuilt -O3 -march=x86-64-v3"


def run_reference_arm(args, world, rank):
    """--impl reference: the reference algorithm on this host's CPU cores."""
    if rank != 0:
        return 0
    sysobj = make_config(args.workload)
    impl, kind, build = pick_cpu_impl(sysobj)
    periodic = sysobj.notes["periodic"]
    threads = os.cpu_count() or 1

    def step():
        H, S = impl.assemble_core(sysobj, periodic)
        if periodic:
            ev = impl.solve_periodic_ops(H, S, threads)
        else:
            ev = impl.solve_box_dense(H.dense, S.dense)
        impl.free(H)
        impl.free(S)
        return ev

    for _ in range(args.warmup):
        step()
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        step()
        times.append((time.perf_counter() - t0) * 1e3)
    ms = float(np.mean(times))
    line = {
        "metric": METRIC, "value": ms, "unit": "ms", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE config, SURVEY.md 8(d))", "impl": "reference",
        "config": workload_config(args.workload, sysobj, world),
        "cpu_baseline": {"value": ms, "unit": "ms", "cores": threads, "kind": kind,
                         "sample": f"full {args.workload} solve per step ({build}; assembly single-threaded as in "
                                   f"the reference; k-point pencils on {threads} threads)"},
        "e2e": {"value": ms, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(workload, budget_s):
    sysobj = make_config(workload)
    impl, kind, build = pick_cpu_impl(sysobj)
    periodic = sysobj.notes["periodic"]
    threads = os.cpu_count() or 1
    times = []
    t_start = time.perf_counter()
    while True:
        t0 = time.perf_counter()
        H, S = impl.assemble_core(sysobj, periodic)
        if periodic:
            impl.solve_periodic_ops(H, S, threads)
        else:
            impl.solve_box_dense(H.dense, S.dense)
        impl.free(H)
        impl.free(S)
        times.append((time.perf_counter() - t0) * 1e3)
        if time.perf_counter() - t_start > budget_s or len(times) >= 50:
            break
    return {"value": float(statistics.median(times)), "unit": "ms", "cores": threads, "kind": kind,
            "sample": f"{len(times)} full {workload} solves (median; {build}); assembly single-threaded like the reference, "
                      f"pencils on {threads} threads; {os.cpu_count()} host cores"}


def chain_system(L):
    """Time-vs-L systems: the reference's gaussian_chain (acceptance_main.cpp:92-103; paper
    Table 1): one nucleus per cell, m0 = 4 s-type functions, n = nbar = 8, M = 8, b = 8."""
    from paper_1408_3839_b200.system import LatticeSystem
    return LatticeSystem(b=8.0, L=(L, 1, 1), n=(8, 8, 8), nbar=(8, 8, 8), quad_M=8, nuc_pos=[(0.0, 0.0, 0.0)],
                         nuc_charge=[1.0], bf_center=[(0.0, 0.0, 0.0)] * 4, bf_alpha=[0.3, 0.5, 0.9, 1.5],
                         name=f"chain{L}")


def scanned(sysobj, i):
    """The i-th point of an exponent scan around `sysobj` (every alpha scaled by 1 + 1e-6 (i+1)):
    a fresh system for the cold end-to-end leg (new plan, new graph, no L0 speculation)."""
    import copy
    s = copy.copy(sysobj)
    s.bf_alpha = np.asarray(sysobj.bf_alpha, dtype=np.float64) * (1.0 + 1e-6 * (i + 1))
    return s


class GpuArm:
    """Device-timed, stage-timed and end-to-end measurement of one workload on this rank."""

    def __init__(self, ctx, dev, world, rank, flush):
        self.ctx, self.dev, self.world, self.rank, self.flush = ctx, dev, world, rank, flush

    def measure(self, workload, steps, warmup, split="kpoints", stages=True, cold=True):
        import torch
        import torch.distributed as dist
        from paper_1408_3839_b200.dist import solve_core_distributed, solve_core_sharded
        ctx, dev, world = self.ctx, self.dev, self.world
        sysobj = make_config(workload)
        periodic = sysobj.notes["periodic"]
        count = sysobj.basis_count
        dsys = ctx.upload(sysobj)
        eig = torch.empty(count, dtype=torch.float64, device=dev)
        ext = torch.cuda.ExternalStream(ctx.stream, device=dev)
        info = np.zeros(8, dtype=np.int64)
        dsys.solve(periodic, eig.data_ptr(), 0, -1, info)  # fills info (L0, bands, R_tot, ...)
        shard_bufs = None
        if world > 1 and split == "rankterms":
            li, _ = dsys.layout(periodic)
            shard_bufs = (torch.empty(int(li[6]), dtype=torch.float64, device=dev),
                          torch.empty(int(li[6]), dtype=torch.float64, device=dev), eig)

        def step():
            if shard_bufs is not None:
                return solve_core_sharded(ctx, sysobj, periodic, dsys=dsys, buffers=shard_bufs)
            return solve_core_distributed(ctx, sysobj, periodic, dsys=dsys, eig_dev=eig, info=info)

        for _ in range(warmup):
            step()
        torch.cuda.synchronize()

        def timed_region(stage_timing):
            ctx.set_stage_timing(stage_timing)
            if stage_timing:
                # the timed graph (event nodes per stage) is captured on the 2nd call: warm it,
                # then reset the totals so only graph replays are counted
                for _ in range(3):
                    step()
                ctx.set_stage_timing(True)
            if world > 1:
                dist.barrier()
            torch.cuda.synchronize()
            l0 = ctx.launches
            ms = []
            for i in range(steps):
                self.flush.fill_(float(i))  # L2 flush between timed iterations (outside the events)
                torch.cuda.synchronize()
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(ext)
                step()
                e1.record(torch.cuda.current_stream(dev))
                e1.synchronize()
                ms.append(e0.elapsed_time(e1))
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            launches = ctx.launches - l0
            st = ctx.stage_times() if stage_timing else {}
            ctx.set_stage_timing(False)
            return ms, launches, st

        clocks = ClockSampler(int(dev.index or 0))
        clocks.start()
        ms, launches, _ = timed_region(False)
        clk = clocks.stop()
        ms_per_step = self._max_over_ranks(sum(ms)) / steps
        stage_tot = {}
        if stages:
            _, _, stage_tot = timed_region(True)

        e2e_out = np.empty(count)  # the caller's result buffer, reused across calls (numpy's out=)

        def e2e_call(s):
            if world == 1:
                return ctx.solve_core(s, periodic, out=e2e_out)
            fn = solve_core_sharded if shard_bufs is not None else solve_core_distributed
            return fn(ctx, s, periodic).cpu().numpy()

        def e2e_leg(systems):
            out = []
            for i, s in enumerate(systems):
                self.flush.fill_(float(i))
                torch.cuda.synchronize()
                if world > 1:
                    dist.barrier()
                t0 = time.perf_counter()
                e2e_call(s)
                out.append((time.perf_counter() - t0) * 1e3)
            return self._max_over_ranks(float(np.mean(out)))

        # end to end through the public API: host LatticeSystem -> host eigenvalues
        # (warm: the same system every step, so the plan and the captured graph are re-used)
        for _ in range(warmup):
            e2e_call(sysobj)
        torch.cuda.synchronize()
        e2e_warm = e2e_leg([sysobj] * steps)
        # cold: a fresh system every step (an exponent scan): planning and eager launches are paid
        # every call
        e2e_cold = e2e_leg([scanned(sysobj, i) for i in range(min(steps, 20))]) if cold else None
        return {"sysobj": sysobj, "periodic": periodic, "info": info.copy(), "ms_per_step": ms_per_step,
                "launches": launches, "clocks": clk, "stages": stage_tot, "e2e_warm": e2e_warm, "e2e_cold": e2e_cold,
                "split": "rankterms" if shard_bufs is not None else "kpoints"}

    def _max_over_ranks(self, v):
        import torch
        import torch.distributed as dist
        t = torch.tensor([float(v)], dtype=torch.float64, device=self.dev)
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())


def roofline_fields(ctx, m, steps, peaks, workload):
    """(dominant-kernel roofline, per-stage table) from the stage-timed pass."""
    sysobj, periodic, stages = m["sysobj"], m["periodic"], m["stages"]
    L0 = int(m["info"][0])
    work = stage_work(ctx, sysobj, periodic, L0)
    per_stage, step_frac = roofline(work, stages, steps, peaks, m["ms_per_step"])
    roof = None
    if stages:
        # dominant kernel by measured time; achieved = its algorithmic amount per launch over
        # its mean launch time (CUDA events on the context stream)
        name, (tot_ms, nl) = max(stages.items(), key=lambda kv: kv[1][0])
        avg_ms = tot_ms / max(1, nl)
        st = per_stage[name]
        if "bound" in st:
            per_launch = st["algorithmic_per_step"] * steps / max(1, nl)
            hbm = st["bound"] == "hbm"
            achieved = per_launch / (avg_ms * 1e-3) / (1e9 if hbm else 1e12)
            peak = st["peak"]
            roof = {"kernel": name, "bound": st["bound"], "achieved": achieved, "peak": peak,
                    "unit": "GB/s" if hbm else "TFLOP/s", "frac": achieved / peak,
                    "traffic": measured_traffic(workload, name),
                    "avg_launch_ms": avg_ms, "launches_per_step": nl / steps,
                    # share of the summed kernel time (comparable with the ncu launch list)
                    "share_of_step": tot_ms / sum(v[0] for v in stages.values()),
                    "algorithmic_per_launch": per_launch,
                    "peak_source": peaks["hbm_src"] if hbm else peaks["fp64_src"],
                    "step_roofline_frac": step_frac}
        else:
            roof = {"kernel": name, "bound": None, "achieved": None, "peak": None, "unit": None, "frac": None,
                    "traffic": None, "avg_launch_ms": avg_ms, "step_roofline_frac": step_frac}
    stage_table = {k: per_stage[k] for k, _ in sorted(stages.items(), key=lambda kv: -kv[1][0])}
    return roof, stage_table


def galerkin_entries(sysobj, periodic, L0):
    bands = [min(L0, sysobj.L[l] - 1) for l in range(3)]
    if periodic:
        nblocks = int(np.prod([2 * b + 1 for b in bands]))
    else:
        nblocks = int(np.prod([sum(1 for k in range(sysobj.L[l]) for d in range(-bands[l], bands[l] + 1)
                                   if 0 <= k + d < sysobj.L[l]) for l in range(3)]))
    return sysobj.m0 ** 2 * nblocks  # Galerkin H entries (S alongside)


def time_vs_L(ctx, reps=5):
    """The metric's 'time vs L': whole path (host LatticeSystem -> host eigenvalues, solve_core)
    for periodic gaussian chains, L = 128 ... 32768 (N_b = 4 L); median of `reps` calls after
    two warm-ups, warm (same system every call)."""
    rows = []
    for L in (128, 512, 2048, 8192, 32768):
        s = chain_system(L)
        for _ in range(2):
            ctx.solve_core(s, True)
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            ctx.solve_core(s, True)
            ts.append((time.perf_counter() - t0) * 1e3)
        rows.append({"L": L, "N_b": 4 * L, "ms": float(np.median(ts))})
    return rows


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="c5", choices=sorted(WORKLOAD_DESC))
    ap.add_argument("--secondary", default="c3", help="extra workload measured into the same line ('' = none)")
    ap.add_argument("--no-sweep", action="store_true", help="skip the time-vs-L rows")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--stages", action="store_true", help="print per-kernel stage times to stderr")
    ap.add_argument("--split", default="kpoints", choices=["kpoints", "rankterms"],
                    help="N > 1: k-point shards with a replicated assembly (default), or the assembly sharded "
                         "by nuclear rank terms with one all-reduce of H, then k-point shards (SURVEY 8(e))")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        return run_reference_arm(args, world, rank)

    import torch
    import torch.distributed as dist
    from paper_1408_3839_b200.api import Context

    if world > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    ctx = Context(local)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2
    arm = GpuArm(ctx, dev, world, rank, flush)
    m = arm.measure(args.workload, args.steps, args.warmup, args.split)
    sec = None
    if args.secondary and args.secondary != args.workload:
        sec = arm.measure(args.secondary, min(args.steps, 20), args.warmup, args.split, cold=False)
    sweep = time_vs_L(ctx) if (not args.no_sweep and world == 1) else None

    if rank == 0:
        peaks = load_peaks()
        sysobj, periodic, info = m["sysobj"], m["periodic"], m["info"]
        L0 = int(info[0])
        ms_per_step = m["ms_per_step"]
        roof, stage_table = roofline_fields(ctx, m, args.steps, peaks, args.workload)
        entries = galerkin_entries(sysobj, periodic, L0)
        cpu = None
        if not args.no_cpu_baseline and world == 1:
            try:
                cpu = cpu_baseline(args.workload, args.cpu_seconds)
            except Exception as e:  # oracle not built on this host
                cpu = {"value": None, "unit": "ms", "cores": 0, "kind": "port", "sample": f"unavailable: {e}"}
        config = workload_config(args.workload, sysobj, world)
        line = {
            "metric": METRIC,
            "value": ms_per_step,
            "unit": "ms",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": False,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f64",
            "data": "synthetic: seeded BASELINE config (splitmix64, SURVEY.md 8(d)); system resident on device",
            "config": config,
            "derived": {"L0": L0, "band": [int(x) for x in info[1:4]], "R_tot": int(info[4]),
                        "N_b": int(info[5]), "k_points": int(info[6]), "split": m["split"]},
            "galerkin_entries_per_s": float(entries) / (ms_per_step * 1e-3) if ms_per_step else None,
            "roofline": roof,
            "stages": stage_table,
            "cpu_baseline": cpu,
            "e2e": {"value": m["e2e_warm"], "unit": "ms", "h2d_bytes_per_step": sysobj.host_bytes(),
                    "d2h_bytes_per_step": 8 * sysobj.basis_count,
                    "what": "host API (LatticeSystem -> host eigenvalues), same system every step: the "
                            "captured graph and plan are re-used"},
            "e2e_cold": {"value": m["e2e_cold"], "unit": "ms",
                         "what": "host API, a fresh system every step (exponent scan, alpha x (1 + 1e-6 i)): "
                                 "planning and eager (uncaptured) launches every call; the lattice-DFT index maps and "
                                 "the L0 prediction carry over between systems of one shape"},
            "gpu_launches": int(m["launches"] / args.steps) * args.steps,
            "gpu_launches_per_step": m["launches"] / args.steps,
            "clocks": m["clocks"],
        }
        if sec is not None:
            sroof, sstages = roofline_fields(ctx, sec, min(args.steps, 20), peaks, args.secondary)
            sl0 = int(sec["info"][0])
            line["secondary"] = {
                "config": workload_config(args.secondary, sec["sysobj"], world),
                "value": sec["ms_per_step"], "unit": "ms", "steps": min(args.steps, 20),
                "e2e": {"value": sec["e2e_warm"], "unit": "ms", "h2d_bytes_per_step": sec["sysobj"].host_bytes(),
                        "d2h_bytes_per_step": 8 * sec["sysobj"].basis_count},
                "galerkin_entries_per_s": galerkin_entries(sec["sysobj"], sec["periodic"], sl0)
                / (sec["ms_per_step"] * 1e-3),
                "roofline": sroof, "stages": sstages, "clocks": sec["clocks"],
                "gpu_launches_per_step": sec["launches"] / min(args.steps, 20)}
        if sweep is not None:
            line["time_vs_L"] = {"what": "whole path (solve_core, host in / host out), periodic gaussian_chain(L) "
                                         "(acceptance_main.cpp:92-103), m0 = 4, median of 5 warm calls",
                                 "rows": sweep}
        print(json.dumps(line), flush=True)
        if args.stages:
            for k, v in sorted(m["stages"].items(), key=lambda kv: -kv[1][0]):
                print(f"  {k:14s} {v[0] / args.steps * 1e3:9.1f} us/step  launches/step {v[1] / args.steps:.1f}",
                      file=sys.stderr)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
