"""Lattice-system description and the seeded BASELINE configurations.

Mirrors ``latham::LatticeSystem`` (reference ``proj/core/include/latham/galerkin.hpp:17-35``)
with the per-direction grid counts of SURVEY.md Appendix B.1 (``n``/``nbar`` are
3-vectors; the reference's scalar ``n`` is the isotropic special case), plus
``NucleiSet`` (``newton_kernel.hpp:12-28``) and ``GtoBasis`` (``gto_basis.hpp:12-29``).

``to_c()`` produces the POD ``lt_system`` of ``include/latham_b200.h`` (the same layout
as the oracle's ``or_system``), keeping the backing arrays alive.
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field
from typing import List, Sequence, Tuple

import numpy as np


class LtSystem(ctypes.Structure):
    """``lt_system`` (include/latham_b200.h)."""

    _fields_ = [
        ("b", ctypes.c_double),
        ("L", ctypes.c_int64 * 3),
        ("n", ctypes.c_int64 * 3),
        ("nbar", ctypes.c_int64 * 3),
        ("quad_M", ctypes.c_int64),
        ("eps_ov", ctypes.c_double),
        ("n_nuclei", ctypes.c_int64),
        ("nuc_pos", ctypes.POINTER(ctypes.c_double)),
        ("nuc_charge", ctypes.POINTER(ctypes.c_double)),
        ("m0", ctypes.c_int64),
        ("bf_center", ctypes.POINTER(ctypes.c_double)),
        ("bf_alpha", ctypes.POINTER(ctypes.c_double)),
        ("bf_deg", ctypes.POINTER(ctypes.c_int32)),
    ]


def _as3(v) -> Tuple[int, int, int]:
    if isinstance(v, (int, np.integer)):
        return (int(v),) * 3
    t = tuple(int(x) for x in v)
    assert len(t) == 3
    return t


@dataclass
class LatticeSystem:
    """Geometry and discretisation of one (L1,L2,L3) lattice system (galerkin.hpp:17-35)."""

    b: float
    L: Tuple[int, int, int]
    n: Tuple[int, int, int]
    nbar: Tuple[int, int, int]
    quad_M: int
    nuc_pos: np.ndarray  # (M0, 3) cell-centred coordinates in [-b/2, b/2]
    nuc_charge: np.ndarray  # (M0,)
    bf_center: np.ndarray  # (m0, 3)
    bf_alpha: np.ndarray  # (m0,)
    bf_deg: np.ndarray = None  # (m0, 3) int32
    eps_ov: float = 1e-8
    name: str = ""
    notes: dict = field(default_factory=dict)

    def __post_init__(self):
        self.L = _as3(self.L)
        self.n = _as3(self.n)
        self.nbar = _as3(self.nbar)
        self.nuc_pos = np.ascontiguousarray(np.asarray(self.nuc_pos, dtype=np.float64).reshape(-1, 3))
        self.nuc_charge = np.ascontiguousarray(np.asarray(self.nuc_charge, dtype=np.float64).reshape(-1))
        self.bf_center = np.ascontiguousarray(np.asarray(self.bf_center, dtype=np.float64).reshape(-1, 3))
        self.bf_alpha = np.ascontiguousarray(np.asarray(self.bf_alpha, dtype=np.float64).reshape(-1))
        if self.bf_deg is None:
            self.bf_deg = np.zeros((len(self.bf_alpha), 3), dtype=np.int32)
        self.bf_deg = np.ascontiguousarray(np.asarray(self.bf_deg, dtype=np.int32).reshape(-1, 3))

    # galerkin.hpp:27-31
    @property
    def m0(self) -> int:
        return int(self.bf_alpha.shape[0])

    @property
    def lattice_count(self) -> int:
        return self.L[0] * self.L[1] * self.L[2]

    @property
    def basis_count(self) -> int:
        return self.m0 * self.lattice_count

    @property
    def rank_N(self) -> int:
        return 2 * self.quad_M + 1

    @property
    def rank_total(self) -> int:
        return self.rank_N * self.nuc_charge.shape[0]

    def h(self, l: int) -> float:
        return self.b / self.n[l]

    def to_c(self) -> LtSystem:
        """The ``lt_system`` view of this object. The struct points at the numpy arrays (in-place
        edits stay visible) and is rebuilt only when a field was re-assigned, so a call with
        the same system does not pay the ctypes marshalling again."""
        key = (self.b, self.L, self.n, self.nbar, self.quad_M, self.eps_ov, id(self.nuc_pos), id(self.nuc_charge),
               id(self.bf_center), id(self.bf_alpha), id(self.bf_deg))
        cached = self.__dict__.get("_c_cache")
        if cached is not None and cached[0] == key:
            return cached[1]
        c = self._build_c()
        self.__dict__["_c_cache"] = (key, c)
        return c

    def _build_c(self) -> LtSystem:
        c = LtSystem()
        c.b = self.b
        for l in range(3):
            c.L[l] = self.L[l]
            c.n[l] = self.n[l]
            c.nbar[l] = self.nbar[l]
        c.quad_M = self.quad_M
        c.eps_ov = self.eps_ov
        c.n_nuclei = self.nuc_charge.shape[0]
        dp = ctypes.POINTER(ctypes.c_double)
        c.nuc_pos = self.nuc_pos.ctypes.data_as(dp)
        c.nuc_charge = self.nuc_charge.ctypes.data_as(dp)
        c.m0 = self.m0
        c.bf_center = self.bf_center.ctypes.data_as(dp)
        c.bf_alpha = self.bf_alpha.ctypes.data_as(dp)
        c.bf_deg = self.bf_deg.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        c._keep = (self.nuc_pos, self.nuc_charge, self.bf_center, self.bf_alpha, self.bf_deg)
        return c

    def host_bytes(self) -> int:
        """Bytes of the host-side system description (the e2e h2d payload)."""
        return int(ctypes.sizeof(LtSystem) + self.nuc_pos.nbytes + self.nuc_charge.nbytes + self.bf_center.nbytes
                   + self.bf_alpha.nbytes + self.bf_deg.nbytes)

    def with_(self, **kw) -> "LatticeSystem":
        d = dict(b=self.b, L=self.L, n=self.n, nbar=self.nbar, quad_M=self.quad_M, nuc_pos=self.nuc_pos,
                 nuc_charge=self.nuc_charge, bf_center=self.bf_center, bf_alpha=self.bf_alpha,
                 bf_deg=self.bf_deg, eps_ov=self.eps_ov, name=self.name, notes=dict(self.notes))
        d.update(kw)
        return LatticeSystem(**d)


# ---------------------------------------------------------------------------
# Seeded inputs: splitmix64, u = (x >> 11) * 2^-53,
# alpha = exp(ln lo + u (ln hi - ln lo)); draw order: nuclei (Z then x), then exponents.
# ---------------------------------------------------------------------------
class SplitMix64:
    MASK = (1 << 64) - 1

    def __init__(self, seed: int):
        self.state = seed & self.MASK

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & self.MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.MASK
        return z ^ (z >> 31)

    def uniform(self) -> float:
        return (self.next_u64() >> 11) * (1.0 / 9007199254740992.0)


SEED_BASE = 0x14083839

# c5's exponent set is rejection-sampled: draw sets in sequence and keep the first
# for which (a) the reference alias guard L_l > 2 L0 (galerkin.cpp:294-302) holds,
# i.e. L0 <= 7, and (b) the reference pencil is definite at every k-point (the
# truncated 3D circulant overlap of near-dependent diffuse pairs can lose
# definiteness; eigensolver.cpp:80-83 then raises DefinitenessError). The accepted
# draw index is fixed here and re-verified by tests/test_configs.py with the oracle.
C5_ACCEPTED_DRAW = 35  # draws 15, 21, 24, 29, 33 pass (a) but fail (b); the rest fail (a)
# c4 (m0 = 16 on 4 nuclei in a 2-bohr cell, alpha down to 0.03) uses rule (b) only:
# draws 0..10 make the reference raise DefinitenessError at some k-point.
C4_ACCEPTED_DRAW = 11
# c3 (box): draw 0 gives an indefinite overlap matrix (lambda_min(S) = -1.6e-6), which
# the reference refuses in solve_box_dense; draw 1 is accepted (rule (b)).
C3_ACCEPTED_DRAW = 1


def _log_uniform(rng: SplitMix64, lo: float, hi: float) -> float:
    return math.exp(math.log(lo) + rng.uniform() * (math.log(hi) - math.log(lo)))


_SPECS = {
    # name: (index, periodic, L, n per cell, m0, (alpha lo, hi), R from the config, nuclei spec)
    "c1": (0, False, (8, 1, 1), (32, 256, 256), 4, (0.1, 10.0), 24, "pair"),
    "c2": (1, True, (32, 1, 1), (32, 256, 256), 8, (0.05, 20.0), 28, "pair"),
    "c3": (2, False, (128, 1, 1), (64, 256, 256), 8, (0.05, 20.0), 32, "pair"),
    "c4": (3, True, (512, 1, 1), (64, 384, 384), 16, (0.03, 30.0), 32, "random4"),
    "c5": (4, True, (16, 16, 16), (64, 64, 64), 8, (0.05, 20.0), 32, "pair"),
}

CONFIG_NAMES = tuple(_SPECS)


def config_periodic(name: str) -> bool:
    return _SPECS[name][1]


def make_config(name: str, exponent_draw: int = None) -> LatticeSystem:
    """Seeded BASELINE.json config `name` mapped per SURVEY.md Appendix B.

    * n per cell: lattice directions split the config's total grid over L cells,
      transverse (L=1) counts are per cell; nbar = n.
    * quad_M = R/2, so the kernel rank is R_N = R+1 (the reference's rank is odd).
    * coordinates are cell-centred: config x = 0.5, 1.5 -> -0.5, +0.5 (b = 2).
    * m0 functions split evenly over the nuclei, centred on them (assumption,
      stated in the bench output).
    """
    idx, periodic, L, n, m0, (alo, ahi), R, nuc_kind = _SPECS[name]
    rng = SplitMix64(SEED_BASE + idx)
    b = 2.0
    if nuc_kind == "pair":
        pos = [(-0.5, 0.0, 0.0), (0.5, 0.0, 0.0)]
        Z = [1.0, 1.0]
    else:
        pos, Z = [], []
        for _ in range(4):
            Z.append(float(1 + min(2, int(rng.uniform() * 3))))
            pos.append((-1.0 + 2.0 * rng.uniform(), 0.0, 0.0))
    per = m0 // len(Z)
    centers = [pos[i // per] for i in range(m0)]
    draw = 0
    if exponent_draw is None:
        exponent_draw = {"c5": C5_ACCEPTED_DRAW, "c4": C4_ACCEPTED_DRAW, "c3": C3_ACCEPTED_DRAW}.get(name, 0)
    alphas = None
    for draw in range(exponent_draw + 1):
        alphas = [_log_uniform(rng, alo, ahi) for _ in range(m0)]
    sysobj = LatticeSystem(b=b, L=L, n=n, nbar=n, quad_M=R // 2, nuc_pos=pos, nuc_charge=Z, bf_center=centers,
                           bf_alpha=alphas, name=name)
    sysobj.notes = {
        "periodic": periodic,
        "seed": hex(SEED_BASE + idx),
        "exponent_draw": exponent_draw,
        "R_config": R,
        "R_N": 2 * (R // 2) + 1,
        "basis_layout": "m0/M0 s-type GTOs per nucleus, centred on it (assumption)",
        "padding": "reference margin L0+2 unit cells (no padding knob in the reference)",
    }
    return sysobj

