"""Algorithmic work per kernel stage.

`stage_work(ctx, sys, periodic, L0)` returns {stage: (bound, amount_per_solve, unit)} with
amounts in bytes ("hbm") or flops ("tensor"), counted from the actual GTO supports the
device computes (lt_profiles), never from the padded tiles a kernel happens to sweep:

- nuclear contraction (triv_gemm, nuc_fold, hankel_gemm): 2 flops per product over the
  exact support intersections dot3 bounds (galerkin.cpp:111-118); symmetric trivial
  tables count mu <= nu only; periodic folds count d >= 0 only (the d < 0 half is a
  mirror). This is the folded count: the reference's redundant work is never credited.
- GEMM reassociations (vgemm, fold_gemm): 2 M N K of the dense product.
- FEM tables (fem_fold): 2 flops x {mass, stiffness} over the pwl support intersections.
- lattice sums / FFT / scatters / pencils / profiles: bytes read + written once (HBM
  lower bound); the batched pencils are latency-bound and reported against HBM as
  SURVEY.md §8(d) asks.
- box dense pencil: potrf N_b^3/3, trsm 2 N_b^3, sytrd (4/3) N_b^3 flops (library sygvd, when
  forced with LT_BOX_SYGVD: (8/3) N_b^3).
"""
from __future__ import annotations

from typing import Dict, Tuple

import numpy as np

KMAX_L0 = 256


def direction_sources(s) -> list:
    """src[l] = first direction with bitwise-identical inputs (engine.cu direction_sources)."""
    src = [0, 1, 2]
    for l in range(1, 3):
        for q in range(l):
            if src[q] != q:
                continue
            if (s.L[q], s.n[q], s.nbar[q]) != (s.L[l], s.n[l], s.nbar[l]):
                continue
            if (np.array_equal(s.nuc_pos[:, q], s.nuc_pos[:, l]) and np.array_equal(s.bf_center[:, q], s.bf_center[:, l])
                    and np.array_equal(s.bf_deg[:, q], s.bf_deg[:, l])):
                src[l] = q
                break
    return src


def _overlap(a0, a1, b0, b1, lo, hi):
    return np.maximum(0, np.minimum(np.minimum(a1, b1), hi) - np.maximum(np.maximum(a0, b0), lo))


def stage_work(ctx, s, periodic: bool, L0: int) -> Dict[str, Tuple[str, float, str]]:
    m0, mm = s.m0, s.m0 * s.m0
    RN, Rtot, nnuc = s.rank_N, s.rank_total, s.nuc_charge.shape[0]
    margin = L0 + 2
    band = [min(L0, s.L[l] - 1) for l in range(3)]
    width = [2 * b + 1 for b in band]
    G = [(s.L[l] + 2 * margin) * s.n[l] for l in range(3)]
    Gbar = [(s.L[l] + 2 * margin) * s.nbar[l] for l in range(3)]
    K = s.lattice_count
    src = direction_sources(s)
    uniq = [l for l in range(3) if src[l] == l]
    prof = ctx.profiles(s, margin)
    sup = {}
    for kind in ("pwc", "pwl"):
        for l in range(3):
            lo = np.array([prof[(kind, l, mu)][0] for mu in range(m0)], dtype=np.int64)
            hi = lo + np.array([len(prof[(kind, l, mu)][1]) for mu in range(m0)], dtype=np.int64)
            sup[(kind, l)] = (lo, hi)
    nblocks = int(np.prod(width)) if periodic else None
    out: Dict[str, Tuple[str, float, str]] = {}

    def add(name, bound, amount, unit):
        if name in out:
            out[name] = (bound, out[name][1] + amount, unit)
        else:
            out[name] = (bound, float(amount), unit)

    # ---- L0
    # s-type directions take the peak-window search (16 profile evaluations per task,
    # latency-bound; counted as its 8-byte result reads), p-type ones sample and scan
    ntask = 0
    for l in uniq:
        if np.all(s.bf_deg[:, l] == 0):
            ntask += (L0 + 2) * m0 * m0
        else:
            lo, hi = sup[("pwc", l)]
            add("l0_sample", "hbm", 8.0 * float(np.sum(hi - lo)), "B")
            add("l0_scan", "hbm", 8.0 * float(np.sum(hi - lo)), "B")
    if ntask:
        add("l0_peak", "hbm", 8.0 * ntask, "B")
    # ---- sinc + lattice-summed potential: master written, master read + windows written
    add("sinc", "hbm", 8.0 * (2 * RN + Rtot), "B")
    for l in uniq:
        wrapped = periodic and s.L[l] > 1
        Lsum = s.L[l] if (wrapped or not periodic) else 1
        if wrapped:
            mrows = s.n[l] + 2 * (s.n[l] * (s.L[l] // 2) + s.n[l])
            rows = s.n[l]
        else:
            NL = s.n[l] * Lsum
            mrows = NL + 2 * margin * s.n[l] + 2 * ((NL + 1) // 2 + s.n[l])
            rows = NL + 2 * margin * s.n[l]
        add("master", "hbm", 8.0 * mrows * RN, "B")
        add("window_sum", "hbm", 8.0 * RN * (mrows + nnuc * rows), "B")
    # ---- profiles (pwc + pwl written)
    add("profiles", "hbm", 8.0 * m0 * sum(G[l] + Gbar[l] for l in uniq), "B")
    # ---- FEM: T v (read v, write two rows) and the tables
    fem_fl = 0.0
    for l in uniq:
        add("fem_apply", "hbm", 8.0 * m0 * 3 * Gbar[l], "B")
        lo, hi = sup[("pwl", l)]
        for d in range(-band[l], band[l] + 1):
            sh = d * s.nbar[l]
            ov = _overlap(lo[:, None], hi[:, None], lo[None, :] + sh, hi[None, :] + sh, -1, Gbar[l] + 1)
            fem_fl += 2.0 * 2.0 * float(ov.sum())
        add("fold_prep", "hbm", 2 * 8.0 * 3 * m0 * Gbar[l], "B")
        add("resfold_reduce", "hbm", 8.0 * 2 * s.nbar[l] * width[l] * mm, "B")
    add("fem_fold", "tensor", fem_fl, "flop")
    # ---- nuclear contraction
    triv = [l for l in uniq if s.L[l] == 1]
    wrapped_dirs = [l for l in range(3) if s.L[l] > 1]
    wrapped_uniq = [l for l in uniq if s.L[l] > 1]
    iu = np.triu_indices(m0)
    for l in triv:
        lo, hi = sup[("pwc", l)]
        rows = G[l]  # open direction: the potential panel spans the extended grid
        ov = _overlap(lo[:, None], hi[:, None], lo[None, :], hi[None, :], 0, rows)
        add("triv_gemm", "tensor", 2.0 * Rtot * float(ov[iu].sum()), "flop")
        add("triv_reduce_w", "hbm", 8.0 * (Rtot * len(iu[0]) + Rtot * mm), "B")
    if len(wrapped_dirs) == 1:
        l = wrapped_dirs[0]
        if periodic:  # potential panel rows contracted by V = W^T P
            rows = s.n[l]
        else:
            rows = s.n[l] * s.L[l] + 2 * margin * s.n[l]
        add("vgemm", "tensor", 2.0 * mm * Rtot * rows, "flop")
        lo, hi = sup[("pwc", l)]
        n = s.n[l]
        if periodic:
            fl = 0.0
            for d in range(0, band[l] + 1):
                ov = _overlap(lo[:, None], hi[:, None], lo[None, :] + d * n, hi[None, :] + d * n, 0, G[l])
                fl += 2.0 * float(ov.sum())
            add("nuc_fold", "tensor", fl, "flop")
            add("fold_prep", "hbm", 2 * 8.0 * 2 * m0 * G[l], "B")
            add("resfold_reduce", "hbm", 8.0 * n * (band[l] + 1) * mm, "B")
        else:
            fl = 0.0
            ks = np.arange(s.L[l])
            for d in range(-band[l], band[l] + 1):
                kk = ks[(ks + d >= 0) & (ks + d < s.L[l])]
                if kk.size == 0:
                    continue
                a0 = lo[:, None, None] + kk[None, None, :] * n
                a1 = hi[:, None, None] + kk[None, None, :] * n
                b0 = lo[None, :, None] + (kk[None, None, :] + d) * n
                b1 = hi[None, :, None] + (kk[None, None, :] + d) * n
                fl += 2.0 * float(_overlap(a0, a1, b0, b1, 0, G[l]).sum())
            add("hankel_gemm", "tensor", fl, "flop")
            add("split_reduce", "hbm", 8.0 * mm * s.L[l] * width[l], "B")
    elif periodic and len(wrapped_dirs) >= 2:
        for l in wrapped_uniq:
            lo, hi = sup[("pwc", l)]
            n = s.n[l]
            fl = 0.0
            for d in range(0, band[l] + 1):
                ov = _overlap(lo[:, None], hi[:, None], lo[None, :] + d * n, hi[None, :] + d * n, 0, G[l])
                fl += 2.0 * float(ov.sum())
            add("nuc_fold", "tensor", fl, "flop")
            add("fold_prep", "hbm", 2 * 8.0 * 2 * m0 * G[l], "B")
            add("fold_gemm", "tensor", 2.0 * Rtot * (band[l] + 1) * mm * n, "flop")
        add("kr_combine", "tensor", 3.0 * Rtot * mm * nblocks, "flop")
    # ---- fill (H and S written)
    if periodic:
        add("fill", "hbm", 8.0 * 2 * nblocks * mm, "B")
    else:
        Nb = s.basis_count
        add("fill", "hbm", 8.0 * 2 * Nb * Nb, "B")
    # ---- spectrum
    if periodic:
        # per transformed axis, H and S: read + write K m0^2 complex (single-axis transforms
        # small enough are fused into the pencil load: no dft_axis stage then)
        add("dft_axis", "hbm", 2 * 2 * 16.0 * K * mm * len(wrapped_dirs), "B")
        # >= 2 wrapped axes: one fused launch reads the stored generating blocks once and
        # writes the K Fourier blocks once, H and S
        add("dft_fused", "hbm", 2 * (8.0 * nblocks * mm + 16.0 * K * mm), "B")
        add("pencil", "hbm", K * (2 * 16.0 * mm + 8.0 * m0), "B")
    else:
        Nb = s.basis_count
        if Nb <= 32:
            add("r2c", "hbm", 2 * (8.0 + 16.0) * Nb * Nb, "B")
            add("pencil", "hbm", 2 * 16.0 * Nb * Nb + 8.0 * Nb, "B")
        else:
            # the B200 dense path (k_dense.cu): Cholesky N^3/3, two triangular solves 2 N^3,
            # tridiagonalisation 4/3 N^3 (dsytd2 count), symmetrisation and the tridiagonal
            # eigenvalues as bytes (latency-bound chains); the library sygvd when forced
            add("potrf", "tensor", Nb ** 3 / 3.0, "flop")
            add("trsm", "tensor", 2.0 * Nb ** 3, "flop")
            add("sytrd", "tensor", (4.0 / 3.0) * Nb ** 3, "flop")
            add("symmetrize", "hbm", 2 * 8.0 * Nb * Nb, "B")
            add("tridiag_eig", "hbm", 8.0 * 3 * Nb, "B")
            add("sygvd", "tensor", (8.0 / 3.0) * Nb ** 3, "flop")
    return out


def roofline(work, stages, steps, peaks, step_ms):
    """Per-stage and whole-step roofline from measured stage times.

    stages: {name: (total_ms, launches)} over `steps` solves. Returns (per_stage, step_frac)
    with step_frac = sum_s max(F_s/P, B_s/BW) / t_step."""
    per = {}
    ideal_ms = 0.0
    for name, (tot_ms, nl) in stages.items():
        ms = tot_ms / steps
        if name not in work:
            per[name] = {"ms_per_step": ms, "launches_per_step": nl / steps}
            continue
        bound, amount, unit = work[name]
        if bound == "hbm":
            peak, ach = peaks["hbm_gbs"], amount / (ms * 1e-3) / 1e9
            ideal = amount / (peak * 1e9) * 1e3
        else:
            peak, ach = peaks["fp64_tflops"], amount / (ms * 1e-3) / 1e12
            ideal = amount / (peak * 1e12) * 1e3
        ideal_ms += ideal
        per[name] = {"ms_per_step": ms, "launches_per_step": nl / steps, "bound": bound,
                     "algorithmic_per_step": amount, "unit": unit, "achieved": ach, "peak": peak,
                     "frac": ach / peak}
    return per, (ideal_ms / step_ms if step_ms else None)
