"""ctypes binding of Oracle-X (oracle/_build/liblatham_oracle.so) and Oracle-R
(oracle/_ref/libref_latham.so, the reference sources compiled in place).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs, never by the product package.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liblatham_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libref_latham.so")
NATIVE_SO = os.path.join(HERE, "_native", "liblatham_oracle.so")

_P = ctypes.POINTER
_d = ctypes.c_double
_i64 = ctypes.c_int64
_dp = _P(ctypes.c_double)
_ip = _P(ctypes.c_int64)

KINDS = {"laplace": 0, "mass": 1, "nuclear": 2}
ERRORS = {1: "DimensionError", 2: "BoundsError", 3: "StructureError", 4: "DefinitenessError",
          5: "ResourceCapError", 6: "Error"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERRORS.get(code, 'Error')}: {msg}")
        self.code = code
        self.kind = ERRORS.get(code, "Error")
        self.msg = msg


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(_ip)


@dataclass
class Operator:
    """AssembledOperator (galerkin.hpp:43-54) materialised as numpy."""

    periodic: bool
    m0: int
    L: tuple
    L0: int
    coefficient_rank: int
    band: tuple
    dense: Optional[np.ndarray] = None  # (Nb, Nb)
    kidx: Optional[np.ndarray] = None  # (nblk, 3), std::map order
    blocks: Optional[np.ndarray] = None  # (nblk, m0, m0) [row, col]
    separable: Optional[list] = None
    _handle: object = None

    def gen_dict(self):
        return {tuple(int(x) for x in k): self.blocks[i] for i, k in enumerate(self.kidx)}


class Oracle:
    def __init__(self, path: str = ORACLE_SO, prefix: str = "or_"):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (make -C oracle)")
        self.lib = lib = ctypes.CDLL(path)
        self.path = path
        p = prefix
        f = lambda name: getattr(lib, p + name)  # noqa: E731
        self._assemble = f("assemble")
        self._assemble.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, _P(ctypes.c_void_p)]
        self._combine = f("combine")
        self._combine.argtypes = [_d, ctypes.c_void_p, _d, ctypes.c_void_p, _P(ctypes.c_void_p)]
        self._free = f("op_free")
        self._free.argtypes = [ctypes.c_void_p]
        self._info = f("op_info")
        self._info.argtypes = [ctypes.c_void_p, _ip]
        self._dense = f("op_dense")
        self._dense.argtypes = [ctypes.c_void_p, _dp]
        self._blocks = f("op_blocks")
        self._blocks.argtypes = [ctypes.c_void_p, _ip, _dp]
        self._sep = getattr(lib, p + "op_separable", None)
        if self._sep is not None:
            self._sep.argtypes = [ctypes.c_void_p, _dp]
        self._solve_ops = f("solve_periodic_ops")
        self._solve_ops.argtypes = [ctypes.c_void_p, ctypes.c_void_p, _i64, _dp]
        self._solve_fact = getattr(lib, p + "solve_periodic_factorized_ops", None)
        if self._solve_fact is not None:
            self._solve_fact.argtypes = [ctypes.c_void_p, ctypes.c_void_p, _i64, _dp]
        self._solve_gen = f("solve_periodic")
        self._solve_gen.argtypes = [_ip, _i64, _i64, _ip, _dp, _i64, _ip, _dp, _i64, _dp]
        self._bdiag = f("block_diagonalize")
        self._bdiag.argtypes = [_ip, _i64, _i64, _ip, _dp, _dp]
        self._box = f("solve_box_dense")
        self._box.argtypes = [_i64, _dp, _dp, _i64, _dp]
        self._pencil = getattr(lib, p + "solve_pencil", None)
        if self._pencil is not None:
            self._pencil.argtypes = [_i64, _dp, _dp, _i64, _dp]
        # eigenvector entries (Oracle-R only: the reference's want_vectors paths)
        self._box_vec = getattr(lib, p + "solve_box_dense_vec", None)
        if self._box_vec is not None:
            self._box_vec.argtypes = [_i64, _dp, _dp, _i64, _dp, _dp]
        self._gen_vec = getattr(lib, p + "solve_periodic_vec", None)
        if self._gen_vec is not None:
            self._gen_vec.argtypes = [_ip, _i64, _i64, _ip, _dp, _i64, _ip, _dp, _i64, _dp, _dp]
        self._recon = getattr(lib, p + "reconstruct_eigenvectors", None)
        if self._recon is not None:
            self._recon.argtypes = [_ip, _i64, _dp, _i64, _dp]
        self._fullvec = getattr(lib, p + "bc_full_eigenvector", None)
        if self._fullvec is not None:
            self._fullvec.argtypes = [_ip, _i64, _dp, _i64, _i64, _dp]
        self._err = f("last_error")
        self._err.restype = ctypes.c_char_p
        self._sinc = getattr(lib, p + "sinc_quadrature", None)
        if self._sinc is not None:
            self._sinc.argtypes = [_i64, _dp, _dp]
        self._l0 = f("overlap_constant")
        self._l0.argtypes = [ctypes.c_void_p]
        self._l0.restype = _i64
        self._pot = getattr(lib, p + "potential", None)
        if self._pot is not None:
            self._pot.argtypes = [ctypes.c_void_p, ctypes.c_int, _i64, _ip, _ip, _dp, _dp, _i64]
        self._aws = getattr(lib, p + "assembled_window_sum", None)
        if self._aws is not None:
            self._aws.argtypes = [_i64, _i64, _dp, _i64, _ip, _i64, _dp]
        self._master = getattr(lib, p + "newton_master_column", None)
        if self._master is not None:
            self._master.argtypes = [_i64, _d, _i64, _dp]
        self._sample = getattr(lib, p + "sample_gto_1d", None)
        if self._sample is not None:
            self._sample.argtypes = [_dp, _d, _P(ctypes.c_int32), ctypes.c_int, _i64, _d, _i64, _i64, _d, _d, _d,
                                     _ip, _dp]
            self._sample.restype = _i64
        self._tri = getattr(lib, p + "tri_form", None)
        if self._tri is not None:
            self._tri.argtypes = [_i64, _i64, _dp, _i64, _i64, _dp, _d, _d]
            self._tri.restype = _d

    def _check(self, rc: int):
        if rc != 0:
            raise OracleError(rc, self._err().decode())

    # ------------------------------------------------------------------
    def _wrap(self, h) -> Operator:
        info = np.zeros(12, dtype=np.int64)
        self._info(h, _iptr(info))
        periodic, m0 = bool(info[0]), int(info[1])
        L = tuple(int(x) for x in info[2:5])
        op = Operator(periodic=periodic, m0=m0, L=L, L0=int(info[5]), coefficient_rank=int(info[6]),
                      band=tuple(int(x) for x in info[9:12]))
        if periodic:
            nblk = int(info[7])
            kidx = np.zeros((nblk, 3), dtype=np.int64)
            blk = np.zeros(nblk * m0 * m0)
            self._blocks(h, _iptr(kidx), _dptr(blk))
            op.kidx = kidx
            op.blocks = blk.reshape(nblk, m0, m0).transpose(0, 2, 1).copy()  # col-major -> [row, col]
        else:
            Nb = int(info[8])
            d = np.zeros(Nb * Nb)
            self._dense(h, _dptr(d))
            op.dense = d.reshape(Nb, Nb).T.copy()
        op._handle = h
        return op

    def assemble(self, sys, periodic: bool, kind: str) -> Operator:
        c = sys.to_c()
        h = ctypes.c_void_p()
        self._check(self._assemble(ctypes.byref(c), int(periodic), KINDS[kind], ctypes.byref(h)))
        return self._wrap(h)

    def combine(self, wa: float, a: Operator, wb: float, b: Operator) -> Operator:
        h = ctypes.c_void_p()
        self._check(self._combine(wa, a._handle, wb, b._handle, ctypes.byref(h)))
        return self._wrap(h)

    def assemble_core(self, sys, periodic: bool):
        """commands.cpp:51-59: H = 0.5 Laplace - Nuclear, S = Mass."""
        lap = self.assemble(sys, periodic, "laplace")
        nuc = self.assemble(sys, periodic, "nuclear")
        H = self.combine(0.5, lap, -1.0, nuc)
        S = self.assemble(sys, periodic, "mass")
        return H, S

    def separable_terms(self, op: Operator):
        """Rank metadata (galerkin.cpp:394-423): list over terms of [level 0, 1, 2]
        (L_l, m0, m0) [row, col] block sequences."""
        L, m0 = op.L, op.m0
        per = (L[0] + L[1] + L[2]) * m0 * m0
        out = np.zeros(max(1, op.coefficient_rank * per))
        self._sep(op._handle, _dptr(out))
        terms = []
        for t in range(op.coefficient_rank):
            at = t * per
            term = []
            for l in range(3):
                n = L[l] * m0 * m0
                term.append(out[at:at + n].reshape(L[l], m0, m0).transpose(0, 2, 1).copy())
                at += n
            terms.append(term)
        return terms

    def free(self, op: Operator):
        if op._handle is not None:
            self._free(op._handle)
            op._handle = None

    def solve_periodic_ops(self, H: Operator, S: Operator, threads: int = 1) -> np.ndarray:
        K = H.L[0] * H.L[1] * H.L[2]
        out = np.zeros(K * H.m0)
        self._check(self._solve_ops(H._handle, S._handle, threads, _dptr(out)))
        return out.reshape(K, H.m0)

    def solve_periodic_factorized_ops(self, H: Operator, S: Operator, threads: int = 1) -> np.ndarray:
        K = H.L[0] * H.L[1] * H.L[2]
        out = np.zeros(K * H.m0)
        self._check(self._solve_fact(H._handle, S._handle, threads, _dptr(out)))
        return out.reshape(K, H.m0)

    def solve_periodic(self, dims, m0, Hgen: dict, Sgen: dict, threads: int = 1) -> np.ndarray:
        def pack(g):
            keys = sorted(g)
            k = np.array(keys, dtype=np.int64).reshape(-1, 3)
            b = np.concatenate([np.asarray(g[key], dtype=np.float64).T.reshape(-1) for key in keys]) if keys else np.zeros(0)
            return len(keys), k, np.ascontiguousarray(b)
        nH, kH, bH = pack(Hgen)
        nS, kS, bS = pack(Sgen)
        d = np.array(dims, dtype=np.int64)
        K = int(np.prod(d))
        out = np.zeros(K * m0)
        self._check(self._solve_gen(_iptr(d), m0, nH, _iptr(kH), _dptr(bH), nS, _iptr(kS), _dptr(bS), threads,
                                    _dptr(out)))
        return out.reshape(K, m0)

    def block_diagonalize(self, dims, m0, gen: dict) -> np.ndarray:
        keys = sorted(gen)
        k = np.array(keys, dtype=np.int64).reshape(-1, 3)
        b = np.ascontiguousarray(np.concatenate([np.asarray(gen[key], dtype=np.float64).T.reshape(-1) for key in keys]))
        d = np.array(dims, dtype=np.int64)
        K = int(np.prod(d))
        out = np.zeros(K * m0 * m0 * 2)
        self._check(self._bdiag(_iptr(d), m0, len(keys), _iptr(k), _dptr(b), _dptr(out)))
        z = out[0::2] + 1j * out[1::2]
        return z.reshape(K, m0, m0).transpose(0, 2, 1).copy()

    def solve_box_dense(self, H: np.ndarray, S: np.ndarray, cap: int = 4096) -> np.ndarray:
        n = H.shape[0]
        Hc = np.asfortranarray(H, dtype=np.float64)
        Sc = np.asfortranarray(S, dtype=np.float64)
        out = np.zeros(n)
        self._check(self._box(n, Hc.ctypes.data_as(_dp), Sc.ctypes.data_as(_dp), cap, _dptr(out)))
        return out

    def solve_box_dense_vectors(self, H: np.ndarray, S: np.ndarray, cap: int = 4096):
        """solve_box_dense(H, S, want_vectors = true): (eigenvalues, eigenvectors [n, n])."""
        n = H.shape[0]
        Hc = np.asfortranarray(H, dtype=np.float64)
        Sc = np.asfortranarray(S, dtype=np.float64)
        out = np.zeros(n)
        vec = np.zeros(max(n * n, 1))
        self._check(self._box_vec(n, Hc.ctypes.data_as(_dp), Sc.ctypes.data_as(_dp), cap, _dptr(out), _dptr(vec)))
        return out, vec[:n * n].reshape(n, n).T.copy()

    def solve_periodic_vectors(self, dims, m0, Hgen: dict, Sgen: dict, threads: int = 1):
        """solve_periodic(gen, gen, want_vectors = true): (eig [K, m0], vec [K, m0, m0])."""
        def pack(g):
            keys = sorted(g)
            k = np.array(keys, dtype=np.int64).reshape(-1, 3)
            b = np.concatenate([np.asarray(g[key], dtype=np.float64).T.reshape(-1) for key in keys]) if keys else np.zeros(0)
            return len(keys), k, np.ascontiguousarray(b)
        nH, kH, bH = pack(Hgen)
        nS, kS, bS = pack(Sgen)
        d = np.array(dims, dtype=np.int64)
        K = int(np.prod(d))
        out = np.zeros(K * m0)
        vec = np.zeros(2 * K * m0 * m0)
        self._check(self._gen_vec(_iptr(d), m0, nH, _iptr(kH), _dptr(bH), nS, _iptr(kS), _dptr(bS), threads,
                                  _dptr(out), _dptr(vec)))
        z = vec[0::2] + 1j * vec[1::2]
        return out.reshape(K, m0), z.reshape(K, m0, m0).transpose(0, 2, 1).copy()

    @staticmethod
    def _pack_vec(vecs: np.ndarray) -> np.ndarray:
        a = np.asarray(vecs, dtype=np.complex128).transpose(0, 2, 1).reshape(-1)
        o = np.empty(2 * a.size)
        o[0::2], o[1::2] = a.real, a.imag
        return o

    def reconstruct_eigenvectors(self, dims, vecs: np.ndarray, cap: int = 4096) -> np.ndarray:
        K, m0, _ = vecs.shape
        N = K * m0
        d = np.array(dims, dtype=np.int64)
        u = self._pack_vec(vecs)
        out = np.zeros(2 * N * N if N <= cap else 2)
        self._check(self._recon(_iptr(d), m0, _dptr(u), cap, _dptr(out)))
        z = out[0::2] + 1j * out[1::2]
        return z.reshape(N, N).T.copy()

    def bc_full_eigenvector(self, dims, vecs: np.ndarray, j: int, m: int) -> np.ndarray:
        K, m0, _ = vecs.shape
        d = np.array(dims, dtype=np.int64)
        u = self._pack_vec(vecs)
        out = np.zeros(2 * K * m0)
        self._check(self._fullvec(_iptr(d), m0, _dptr(u), j, m, _dptr(out)))
        return out[0::2] + 1j * out[1::2]

    def solve_pencil(self, Hj: np.ndarray, Sj: np.ndarray, j: int = 0) -> np.ndarray:
        m0 = Hj.shape[0]
        def pack(a):
            a = np.asarray(a, dtype=np.complex128).T.reshape(-1)
            o = np.empty(2 * a.size)
            o[0::2], o[1::2] = a.real, a.imag
            return o
        h, s = pack(Hj), pack(Sj)
        out = np.zeros(m0)
        self._check(self._pencil(m0, _dptr(h), _dptr(s), j, _dptr(out)))
        return out

    def sinc_quadrature(self, M: int):
        t = np.zeros(2 * M + 1)
        w = np.zeros(2 * M + 1)
        self._sinc(M, _dptr(t), _dptr(w))
        return t, w

    def overlap_constant(self, sys) -> int:
        c = sys.to_c()
        return int(self._l0(ctypes.byref(c)))

    def potential(self, sys, periodic: bool, margin: int):
        c = sys.to_c()
        rows = np.zeros(3, dtype=np.int64)
        tiled = np.zeros(3, dtype=np.int64)
        self._check(self._pot(ctypes.byref(c), int(periodic), margin, _iptr(rows), _iptr(tiled), None, None, 0))
        R = sys.rank_total
        total = int(rows.sum()) * R
        panels = np.zeros(total)
        w = np.zeros(R)
        self._check(self._pot(ctypes.byref(c), int(periodic), margin, _iptr(rows), _iptr(tiled), _dptr(panels),
                              _dptr(w), total))
        out, at = [], 0
        for l in range(3):
            r = int(rows[l])
            out.append(panels[at:at + r * R].reshape(R, r).T.copy())  # (rows, R)
            at += r * R
        return out, w, tuple(bool(x) for x in tiled)

    def assembled_window_sum(self, master: np.ndarray, shifts, size: int) -> np.ndarray:
        mrows, R = master.shape
        m = np.asfortranarray(master, dtype=np.float64)
        sh = np.array(shifts, dtype=np.int64)
        out = np.zeros(size * R)
        self._check(self._aws(mrows, R, m.ctypes.data_as(_dp), len(sh), _iptr(sh), size, _dptr(out)))
        return out.reshape(R, size).T.copy()

    def newton_master_column(self, ncells: int, h: float, M: int) -> np.ndarray:
        R = 2 * M + 1
        out = np.zeros(ncells * R)
        self._master(ncells, h, M, _dptr(out))
        return out.reshape(R, ncells).T.copy()

    def sample_gto_1d(self, center, alpha, deg, direction, grid_n, step, cell_index, per_cell, b, align, eps):
        c = np.array(center, dtype=np.float64)
        dg = np.array(deg, dtype=np.int32)
        off = np.zeros(1, dtype=np.int64)
        vals = np.zeros(grid_n)
        ln = self._sample(_dptr(c), alpha, dg.ctypes.data_as(_P(ctypes.c_int32)), direction, grid_n, step,
                          cell_index, per_cell, b, align, eps, _iptr(off), _dptr(vals))
        return int(off[0]), vals[:ln].copy()

    def tri_form(self, uoff, u, voff, v, lo, diag) -> float:
        u = np.ascontiguousarray(u, dtype=np.float64)
        v = np.ascontiguousarray(v, dtype=np.float64)
        return float(self._tri(uoff, len(u), _dptr(u), voff, len(v), _dptr(v), lo, diag))


_cache = {}


def oracle() -> Oracle:
    if "x" not in _cache:
        _cache["x"] = Oracle(ORACLE_SO, "or_")
    return _cache["x"]


def reference() -> Optional[Oracle]:
    """Oracle-R (reference sources compiled in place), or None if not built."""
    if "r" not in _cache:
        _cache["r"] = Oracle(REF_SO, "ref_") if os.path.exists(REF_SO) else None
    return _cache["r"]


def native_oracle() -> Optional[Oracle]:
    """Oracle-X built on THIS host with -O3 -march=native (the reference's build flags,
    BASELINE.md), for the CPU baseline; None if the compiler is unavailable."""
    if "n" not in _cache:
        import subprocess
        r = subprocess.run(["make", "-s", "-C", HERE, "native"], capture_output=True, text=True)
        _cache["n"] = Oracle(NATIVE_SO, "or_") if r.returncode == 0 and os.path.exists(NATIVE_SO) else None
    return _cache["n"]
