"""Turn a round's raw ncu output (gpurun_out/prof/) into the committed summaries (profiles/).

    python tools/summarize_profiles.py r01

Writes, per round R:
  profiles/R_<cfg>_launches.csv        every launch: id, kernel, device time (us) — the
                                       `--metrics gpu__time_duration.sum --clock-control none`
                                       pass of the bench command (cold-cache, serialised)
  profiles/R_<cfg>_launch_summary.txt  per-kernel time per solve and share of kernel time
  profiles/R_<cfg>_full_metrics.csv    `--set full` capture: per launch duration, grid,
                                       registers, DRAM bytes, SM / FP64 / DMMA pipe
                                       utilisation, L2 hit rate, top stall reasons
  profiles/R_traffic.json              DRAM bytes per launch by bench stage (roofline.traffic)
  profiles/R_bench.json                the default bench line of the same job
"""
import collections
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "gpurun_out", "prof")
DST = os.path.join(ROOT, "profiles")

# kernel -> bench stage (engine Stage names)
STAGE = {
    "k_pencil": "pencil", "k_l0_scan": "l0_scan", "k_l0_sample": "l0_sample", "k_l0_init": "l0_init",
    "k_triv_gemm": "triv_gemm", "k_triv_reduce_w": "triv_reduce_w", "k_dft_axis2": "dft_axis", "k_dft_fused": "dft_fused", "k_fill": "fill",
    "k_master": "master", "k_window_sum_uniform": "window_sum", "k_window_copy": "window_sum",
    "k_resfold_prep": "fold_prep", "k_resfold_reduce": "resfold_reduce", "k_fem_apply": "fem_apply",
    "k_profile_sample": "profiles", "k_profile_trim": "profiles", "k_sinc": "sinc", "k_hankel": "hankel_gemm",
    "k_split_reduce": "split_reduce", "k_fgemm": "fold_gemm", "k_kr_combine": "kr_combine",
    "k_vgemm": "vgemm", "k_real_to_complex": "r2c", "k_sytrd_reg": "sytrd", "k_sytrd": "sytrd",
    "k_tridiag_eig3": "tridiag_eig", "k_symmetrize": "symmetrize", "k_trtri_leaf": "trtri_leaf",
    "k_l0_peak": "l0_peak", "k_profiles": "profiles", "k_window_sum_short": "window_sum",
    "k_window_sum_staged": "window_sum", "k_hankel_res": "hankel_gemm", "k_split_reduce_quota": "split_reduce",
    "k_pencil_lane": "pencil", "k_potf_leaf": "potf_leaf", "k_vdot": "vdot", "k_resfold": "nuc_fold",
}

FULL_METRICS = [
    ("duration_us", "gpu__time_duration.sum"),
    ("grid", "launch__grid_size"),
    ("block", "launch__block_size"),
    ("regs", "launch__registers_per_thread"),
    ("dram_read_B", "dram__bytes_read.sum"),
    ("dram_write_B", "dram__bytes_write.sum"),
    ("sm_throughput_pct", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
    ("warps_active_pct", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("fp64_pipe_pct", "TPC.TriageCompute.sm__pipe_fp64_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    ("tensor_pipe_pct", "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
    ("l2_hit_pct", "lts__t_sector_hit_rate.pct"),
    ("stall_long_scoreboard", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
    ("stall_barrier", "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio"),
    ("stall_short_scoreboard", "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"),
    ("stall_wait", "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"),
    ("sm_mhz", "smsp__cycles_elapsed.avg.per_second"),
]


def short(name):
    n = name.split("(")[0].replace("void ", "").strip()
    return n.replace("lt::", "")


def base(name):
    return short(name).split("<")[0]


def launches(cfg, R):
    src = os.path.join(SRC, f"{R}_{cfg}_launches.csv")
    if not os.path.exists(src):
        return None
    rows = list(csv.reader(open(src)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    hdr, data = rows[hi], rows[hi + 1:]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    out = []
    for r in data:
        if len(r) <= vi:
            continue
        out.append((int(r[0]), short(r[ki]), float(r[vi].replace(",", "")) / 1e3))
    with open(os.path.join(DST, f"{R}_{cfg}_launches.csv"), "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["id", "kernel", "device_us"])
        w.writerows(out)
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for _, k, us in out:
        tot[k] += us
        cnt[k] += 1
    ours = {k: v for k, v in tot.items() if k.startswith("k_") or "cusolver" in k or "sytrd" in k or "gemm" in k
            or "trsm" in k or "laed" in k or "potrf" in k or "getrf" in k}
    per = max((cnt[k] for k in cnt if k.startswith("k_pencil")), default=0) or \
        max((cnt[k] for k in cnt if k.startswith("k_triv_reduce_w")), default=1)
    s = sum(ours.values())
    lines = [f"{R} {cfg}: {len(out)} launches, {per} solves (normalised by the once-per-solve kernel); "
             f"kernel time per solve {s / per:.1f} us (ncu: cold caches, serialised, clocks not locked)"]
    for k, v in sorted(ours.items(), key=lambda kv: -kv[1]):
        lines.append(f"  {k:60s} {v / per:9.1f} us/solve  {cnt[k] / per:5.1f} launches  share {v / s:.3f}")
    open(os.path.join(DST, f"{R}_{cfg}_launch_summary.txt"), "w").write("\n".join(lines) + "\n")
    print("\n".join(lines[:12]))
    return out


def full(cfg, R, traffic):
    rep = os.path.join(SRC, f"{R}_{cfg}_full.ncu-rep")
    if not os.path.exists(rep):
        return
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    ki = hdr.index("Kernel Name")
    cols = [(lab, hdr.index(m) if m in hdr else None) for lab, m in FULL_METRICS]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
             "usecond": 1.0, "nsecond": 1e-3, "msecond": 1e3, "us": 1.0, "ns": 1e-3, "ms": 1e3}
    out = []
    for r in rows[2:]:
        rec = {"kernel": short(r[ki])}
        for lab, i in cols:
            v = r[i] if i is not None and i < len(r) else ""
            v = v.replace(",", "")
            unit = rows[1][i] if i is not None else ""
            if lab in ("dram_read_B", "dram_write_B", "duration_us") and v:
                try:
                    v = repr(float(v) * scale.get(unit, 1.0))
                except ValueError:
                    pass
            rec[lab] = v
        out.append(rec)
        b = base(r[ki])
        st = STAGE.get(b)
        try:
            tb = float(rec["dram_read_B"] or 0) + float(rec["dram_write_B"] or 0)
        except ValueError:
            tb = None
        if st and tb is not None:
            traffic.setdefault(cfg[:2], {}).setdefault(st, []).append({"kernel": rec["kernel"], "dram_bytes": tb})  # c3b -> c3
    with open(os.path.join(DST, f"{R}_{cfg}_full_metrics.csv"), "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=["kernel"] + [lab for lab, _ in FULL_METRICS])
        w.writeheader()
        w.writerows(out)
    units = {lab: rows[1][i] for lab, i in cols if i is not None}
    open(os.path.join(DST, f"{R}_{cfg}_full_units.json"), "w").write(json.dumps(units, indent=1) + "\n")
    print(f"{cfg}: {len(out)} launches with full sections")


def main():
    R = sys.argv[1] if len(sys.argv) > 1 else "r01"
    os.makedirs(DST, exist_ok=True)
    for cfg in ("c1", "c2", "c3", "c4", "c5"):
        launches(cfg, R)
    traffic = {}
    for cfg in ("c1", "c2", "c3", "c3b", "c4", "c5"):  # c3b: the c3 kernels outside the Cholesky chain
        full(cfg, R, traffic)
    # per stage: mean DRAM bytes per launch
    agg = {cfg: {st: {"dram_bytes_per_launch": sum(x["dram_bytes"] for x in v) / len(v), "launches": len(v),
                      "kernels": sorted({x["kernel"] for x in v})} for st, v in d.items()}
           for cfg, d in traffic.items()}
    open(os.path.join(DST, f"{R}_traffic.json"), "w").write(json.dumps(agg, indent=1) + "\n")
    for name in ("bench.json", "table1.json"):
        b = os.path.join(SRC, f"{R}_{name}")
        if os.path.exists(b) and os.path.getsize(b) > 0:
            shutil.copy(b, os.path.join(DST, f"{R}_{name}"))


if __name__ == "__main__":
    main()
