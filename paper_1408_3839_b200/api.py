"""Host-side mirror of the reference's C++ API for the hot path, backed by the B200 engine.

Same names, argument meaning and error classes as ``proj/core/include/latham``:

========================================  ==================================================
this module                               reference
========================================  ==================================================
``assemble_box(sys, kind)``               ``galerkin.hpp:70``
``assemble_periodic(sys, kind)``          ``galerkin.hpp:74``
``combine(wa, a, wb, b)``                 ``eigensolver.hpp:23-24``
``assemble_core(sys, periodic)``          ``tools/commands.cpp:51-59`` (fused on the device)
``solve_periodic(H, S)``                  ``eigensolver.hpp:29-33``
``solve_box_dense(H, S, cap, want_vectors)`` ``eigensolver.hpp:17-18`` (DenseSpectrum with vectors)
``reconstruct_eigenvectors(spec, cap)``   ``eigensolver.hpp`` (reconstruct_eigenvectors)
``bc_full_eigenvector(spec, j, m)``       ``block_circulant.hpp`` (bc_full_eigenvector)
``bc_block_diagonalize(dims, m0, gen)``   ``block_circulant.hpp:86``
``build_sinc_quadrature(M)``              ``sinc_quadrature.hpp:35``
``overlap_constant(sys)``                 ``gto_basis.hpp:74``
``newton_master(ncells, h, M)``           ``newton_kernel.hpp:35-36`` (one direction)
``potential(sys, periodic, margin)``      ``galerkin.cpp:151-198`` (lattice_potential_*)
``assembled_window_sum(m, shifts, n)``    ``canonical_tensor.hpp:97-99`` (one direction)
``profiles(sys, margin)``                 ``gto_basis.hpp:47-49`` (assembly grids)
``solve_core(sys, periodic)``             assemble_core + solve_* (the whole hot path)
========================================  ==================================================

Everything here calls through the C-ABI of ``include/latham_b200.h``; there is no
CPU computation and no fallback.
"""
from __future__ import annotations

import contextlib
import ctypes
from dataclasses import dataclass
from typing import Dict, Optional, Tuple

import numpy as np

from . import native
from .native import (BoundsError, DefinitenessError, DimensionError, Error, ResourceCapError,  # noqa: F401
                     StructureError, check)
from .system import LatticeSystem

KINDS = {"laplace": 0, "mass": 1, "nuclear": 2}

_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int64)


def _d(a: np.ndarray):
    return a.ctypes.data_as(_dp)


def _i(a: np.ndarray):
    return a.ctypes.data_as(_ip)


@dataclass
class Operator:
    """AssembledOperator (galerkin.hpp:43-54); payload lives on the device."""

    ctx: "Context"
    handle: int
    periodic: bool
    m0: int
    L: Tuple[int, int, int]
    overlap_L0: int
    coefficient_rank: int
    stored: int
    Nb: int
    band: Tuple[int, int, int]

    def dense(self) -> np.ndarray:
        out = np.zeros(self.Nb * self.Nb)
        check(native.lib().lt_op_dense(self.handle, _d(out)))
        return out.reshape(self.Nb, self.Nb).T  # column-major data: a Fortran-ordered view, no copy

    def blocks(self):
        """(kidx (n,3), blocks (n, m0, m0) [row, col]) in std::map order."""
        k = np.zeros((self.stored, 3), dtype=np.int64)
        b = np.zeros(self.stored * self.m0 * self.m0)
        check(native.lib().lt_op_blocks(self.handle, _i(k), _d(b)))
        return k, b.reshape(self.stored, self.m0, self.m0).transpose(0, 2, 1).copy()

    def gen_dict(self) -> Dict[tuple, np.ndarray]:
        k, b = self.blocks()
        return {tuple(int(x) for x in kk): b[i] for i, kk in enumerate(k)}

    def separable(self):
        """Rank metadata (galerkin.hpp:52): list over terms of [level 0, 1, 2] sequences,
        each an (L_l, m0, m0) array of [row, col] blocks (SeparableTerm::level_blocks)."""
        n = int(native.lib().lt_op_separable_count(self.handle))
        out = np.zeros(max(n, 1))
        check(native.lib().lt_op_separable(self.handle, _d(out)))
        return unpack_terms(out[:n], self.L, self.m0)

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                native.lib().lt_op_free(self.handle)
            except Exception:
                pass
            self.handle = None


def pack_terms(terms, L, m0) -> np.ndarray:
    """[t][level][L_l][m0*m0] column-major blocks (the C-ABI term-list layout)."""
    parts = []
    for term in terms:
        for l in range(3):
            seq = np.asarray(term[l], dtype=np.float64).reshape(L[l], m0, m0)
            parts.append(np.ascontiguousarray(seq.transpose(0, 2, 1)).reshape(-1))
    return np.ascontiguousarray(np.concatenate(parts)) if parts else np.zeros(1)


def unpack_terms(flat: np.ndarray, L, m0):
    per = (L[0] + L[1] + L[2]) * m0 * m0
    out = []
    for t in range(flat.size // per if per else 0):
        at = t * per
        term = []
        for l in range(3):
            n = L[l] * m0 * m0
            term.append(flat[at:at + n].reshape(L[l], m0, m0).transpose(0, 2, 1).copy())
            at += n
        out.append(term)
    return out


@dataclass
class DenseSpectrum:
    """DenseSpectrum (eigensolver.hpp): ascending eigenvalues, S-orthonormal eigenvector
    columns (None unless requested)."""

    eigenvalues: np.ndarray
    eigenvectors: Optional[np.ndarray] = None


@dataclass
class KPointSpectrum:
    """KPointSpectrum (spectrum.hpp): per-k ascending eigenvalues [K, m0] and, when
    requested, per-k eigenvector blocks [K, m0, m0] (columns u_{j,m})."""

    dims: Tuple[int, int, int]
    m0: int
    eigenvalues: np.ndarray
    eigenvectors: Optional[np.ndarray] = None
    solver_path: str = "periodic_fft"

    def k_count(self) -> int:
        return int(self.dims[0] * self.dims[1] * self.dims[2])

    def has_vectors(self) -> bool:
        return self.eigenvectors is not None

    def k_multi(self, lin: int):
        d = self.dims
        return (lin // (d[1] * d[2]), (lin // d[2]) % d[1], lin % d[2])

    def sorted_all(self) -> np.ndarray:
        return np.sort(self.eigenvalues.reshape(-1))


def _cvec_out(n: int) -> np.ndarray:
    return np.zeros(2 * n)


def _cblocks(flat: np.ndarray, K: int, m0: int) -> np.ndarray:
    """C-ABI complex column-major blocks -> (K, m0, m0) [row, col]."""
    z = flat[0::2] + 1j * flat[1::2]
    return z.reshape(K, m0, m0).transpose(0, 2, 1).copy()


def _cblocks_in(blocks: np.ndarray) -> np.ndarray:
    a = np.asarray(blocks, dtype=np.complex128).transpose(0, 2, 1).reshape(-1)
    o = np.empty(2 * a.size)
    o[0::2], o[1::2] = a.real, a.imag
    return o


class Context:
    """One GPU: stream, solver handle and cached device buffers (lt_ctx)."""

    def __init__(self, device: int = 0):
        self.lib = native.lib()
        h = ctypes.c_void_p()
        check(self.lib.lt_create(device, ctypes.byref(h)))
        self.h = h
        self.device = device

    def close(self):
        if self.h:
            self.lib.lt_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def torch_device(self):
        """torch.device of this context's GPU (where DeviceSystem buffers live)."""
        import torch
        return torch.device("cuda", self.device)

    @property
    def stream(self) -> int:
        return int(self.lib.lt_stream(self.h) or 0)

    @property
    def launches(self) -> int:
        return int(self.lib.lt_launch_count(self.h))

    def set_stage_timing(self, on: bool):
        check(self.lib.lt_set_stage_timing(self.h, int(on)))

    def set_diagnostics(self, phase_timing: bool = False, host_timing: bool = False):
        """Phase events between graph launches / host-side timestamps (diagnostic tools only)."""
        check(self.lib.lt_set_diagnostics(self.h, (1 if phase_timing else 0) | (2 if host_timing else 0)))

    def stage_timeline(self):
        """[(name, stream, t0_ms, t1_ms)] of the last solve run with stage timing on."""
        n = int(self.lib.lt_stage_timeline_count(self.h))
        out = []
        buf = ctypes.create_string_buffer(128)
        st = ctypes.c_int()
        t0 = ctypes.c_double()
        t1 = ctypes.c_double()
        for i in range(n):
            check(self.lib.lt_stage_timeline_get(self.h, i, buf, 128, ctypes.byref(st), ctypes.byref(t0),
                                                 ctypes.byref(t1)))
            out.append((buf.value.decode(), st.value, t0.value, t1.value))
        return out

    def stage_times(self) -> Dict[str, Tuple[float, int]]:
        """{kernel stage: (total ms, launches)} from CUDA events on the context stream."""
        out = {}
        n = int(self.lib.lt_stage_count(self.h))
        buf = ctypes.create_string_buffer(128)
        ms = ctypes.c_double()
        cnt = ctypes.c_int64()
        for i in range(n):
            check(self.lib.lt_stage_get(self.h, i, buf, 128, ctypes.byref(ms), ctypes.byref(cnt)))
            out[buf.value.decode()] = (ms.value, cnt.value)
        return out

    # ------------------------------------------------------------------
    def _wrap(self, h) -> Operator:
        info = np.zeros(12, dtype=np.int64)
        self.lib.lt_op_info(h, _i(info))
        return Operator(ctx=self, handle=h.value if hasattr(h, "value") else h, periodic=bool(info[0]),
                        m0=int(info[1]), L=tuple(int(x) for x in info[2:5]), overlap_L0=int(info[5]),
                        coefficient_rank=int(info[6]), stored=int(info[7]), Nb=int(info[8]),
                        band=tuple(int(x) for x in info[9:12]))

    def assemble(self, sys: LatticeSystem, periodic: bool, kind: str) -> Operator:
        c = sys.to_c()
        h = ctypes.c_void_p()
        check(self.lib.lt_assemble(self.h, ctypes.byref(c), int(periodic), KINDS[kind], ctypes.byref(h)))
        return self._wrap(h)

    def assemble_box(self, sys: LatticeSystem, kind: str) -> Operator:
        return self.assemble(sys, False, kind)

    def assemble_periodic(self, sys: LatticeSystem, kind: str) -> Operator:
        return self.assemble(sys, True, kind)

    def assemble_core(self, sys: LatticeSystem, periodic: bool) -> Tuple[Operator, Operator]:
        c = sys.to_c()
        h, s = ctypes.c_void_p(), ctypes.c_void_p()
        check(self.lib.lt_assemble_core(self.h, ctypes.byref(c), int(periodic), ctypes.byref(h), ctypes.byref(s)))
        return self._wrap(h), self._wrap(s)

    def combine(self, wa: float, a: Operator, wb: float, b: Operator) -> Operator:
        h = ctypes.c_void_p()
        check(self.lib.lt_combine(self.h, wa, a.handle, wb, b.handle, ctypes.byref(h)))
        return self._wrap(h)

    # ------------------------------------------------------------------
    def solve_core(self, sys: LatticeSystem, periodic: bool, info: Optional[np.ndarray] = None,
                   out: Optional[np.ndarray] = None) -> np.ndarray:
        """LatticeSystem -> eigenvalues on the host ([K, m0] periodic, [N_b] box). ``out``: a
        C-contiguous float64 array of basis_count entries to receive them (numpy's ``out=``
        convention: a buffer reused across calls skips the allocation and its page faults)."""
        c = sys.to_c()
        if out is None:
            out = np.empty(sys.basis_count)
        elif out.dtype != np.float64 or out.size != sys.basis_count or not out.flags.c_contiguous:
            raise ValueError("solve_core: out must be a C-contiguous float64 array of basis_count entries")
        inf = np.zeros(8, dtype=np.int64) if info is None else info
        check(self.lib.lt_solve_core(self.h, ctypes.byref(c), int(periodic), _d(out), _i(inf)))
        return out.reshape(sys.lattice_count, sys.m0) if periodic else out.reshape(-1)

    def upload(self, sys: LatticeSystem) -> "DeviceSystem":
        return DeviceSystem(self, sys)

    def solve_periodic(self, H: Operator, S: Operator, want_vectors: bool = False):
        """solve_periodic (eigensolver.hpp:32-33): [K, m0] eigenvalues, or with want_vectors
        the KPointSpectrum carrying the per-k eigenvector blocks."""
        K = H.L[0] * H.L[1] * H.L[2]
        out = np.zeros(K * H.m0)
        if not want_vectors:
            check(self.lib.lt_solve_periodic_ops(self.h, H.handle, S.handle, _d(out)))
            return out.reshape(K, H.m0)
        vec = _cvec_out(K * H.m0 * H.m0)
        check(self.lib.lt_solve_periodic_ops_vectors(self.h, H.handle, S.handle, _d(out), _d(vec)))
        return KPointSpectrum(tuple(H.L), H.m0, out.reshape(K, H.m0), _cblocks(vec, K, H.m0))

    def solve_periodic_gen(self, dims, m0: int, Hgen: dict, Sgen: dict, want_vectors: bool = False):
        def pack(g):
            keys = sorted(g)
            k = np.ascontiguousarray(np.array(keys, dtype=np.int64).reshape(-1, 3))
            b = np.ascontiguousarray(np.concatenate([np.asarray(g[kk], dtype=np.float64).T.reshape(-1) for kk in keys])
                                     if keys else np.zeros(1))
            return len(keys), k, b
        nH, kH, bH = pack(Hgen)
        nS, kS, bS = pack(Sgen)
        d = np.array(dims, dtype=np.int64)
        K = int(np.prod(d))
        out = np.zeros(K * m0)
        if not want_vectors:
            check(self.lib.lt_solve_periodic(self.h, _i(d), m0, nH, _i(kH), _d(bH), nS, _i(kS), _d(bS), _d(out)))
            return out.reshape(K, m0)
        vec = _cvec_out(K * m0 * m0)
        check(self.lib.lt_solve_periodic_vectors(self.h, _i(d), m0, nH, _i(kH), _d(bH), nS, _i(kS), _d(bS), _d(out),
                                                 _d(vec)))
        return KPointSpectrum(tuple(int(x) for x in dims), m0, out.reshape(K, m0), _cblocks(vec, K, m0))

    def box_circulant_defect(self, sys: LatticeSystem, want_defect: bool = False):
        """box_circulant_defect (galerkin.cpp:445-454): relative Frobenius norm of the box
        nuclear matrix minus the dense periodic circulant (and the defect matrix)."""
        c = sys.to_c()
        r = ctypes.c_double()
        Nb = sys.basis_count
        out = np.zeros(Nb * Nb) if want_defect else None
        check(self.lib.lt_box_circulant_defect(self.h, ctypes.byref(c), ctypes.byref(r),
                                               _d(out) if want_defect else None))
        return (r.value, out.reshape(Nb, Nb).T.copy()) if want_defect else r.value

    # ---- separable metadata / factorized path --------------------------------
    def separable_residual(self, op: Operator) -> float:
        r = ctypes.c_double()
        check(self.lib.lt_separable_residual(self.h, op.handle, ctypes.byref(r)))
        return r.value

    def solve_periodic_factorized(self, H: Operator, S: Operator, metadata_tol: float = 1e-10,
                                  want_vectors: bool = False):
        """solve_periodic_factorized (eigensolver.hpp): [K, m0] eigenvalues (KPointSpectrum
        with the eigenvector blocks when want_vectors)."""
        K = H.L[0] * H.L[1] * H.L[2]
        out = np.zeros(K * H.m0)
        if not want_vectors:
            check(self.lib.lt_solve_periodic_factorized(self.h, H.handle, S.handle, metadata_tol, _d(out)))
            return out.reshape(K, H.m0)
        vec = _cvec_out(K * H.m0 * H.m0)
        check(self.lib.lt_solve_periodic_factorized_vectors(self.h, H.handle, S.handle, metadata_tol, _d(out),
                                                            _d(vec)))
        return KPointSpectrum(tuple(H.L), H.m0, out.reshape(K, H.m0), _cblocks(vec, K, H.m0), "periodic_factorized")

    def factorized_block_diagonalize(self, levels: int, dims, m0: int, terms) -> np.ndarray:
        """factorized_block_diagonalize (factorized_diag.hpp): (K, m0, m0) complex blocks."""
        d = np.array(dims, dtype=np.int64)
        K = int(np.prod(d))
        flat = pack_terms(terms, dims, m0)
        out = np.zeros(K * m0 * m0 * 2)
        check(self.lib.lt_factorized_block_diagonalize(self.h, levels, _i(d), m0, len(terms), _d(flat), _d(out)))
        z = out[0::2] + 1j * out[1::2]
        return z.reshape(K, m0, m0).transpose(0, 2, 1).copy()

    def solve_periodic_factorized_gen(self, dims, m0: int, Hgen: dict, Sgen: dict, Hterms, Sterms,
                                      metadata_tol: float = 1e-10) -> np.ndarray:
        def pack(g):
            keys = sorted(g)
            k = np.ascontiguousarray(np.array(keys, dtype=np.int64).reshape(-1, 3))
            b = np.ascontiguousarray(np.concatenate([np.asarray(g[kk], dtype=np.float64).T.reshape(-1) for kk in keys])
                                     if keys else np.zeros(1))
            return len(keys), k, b
        nH, kH, bH = pack(Hgen)
        nS, kS, bS = pack(Sgen)
        d = np.array(dims, dtype=np.int64)
        K = int(np.prod(d))
        tH = pack_terms(Hterms, dims, m0)
        tS = pack_terms(Sterms, dims, m0)
        out = np.zeros(K * m0)
        check(self.lib.lt_solve_periodic_factorized_gen(self.h, _i(d), m0, nH, _i(kH), _d(bH), len(Hterms), _d(tH),
                                                        nS, _i(kS), _d(bS), len(Sterms), _d(tS), metadata_tol,
                                                        _d(out)))
        return out.reshape(K, m0)

    def bc_block_diagonalize(self, dims, m0: int, gen: dict) -> np.ndarray:
        keys = sorted(gen)
        k = np.ascontiguousarray(np.array(keys, dtype=np.int64).reshape(-1, 3))
        b = np.ascontiguousarray(np.concatenate([np.asarray(gen[kk], dtype=np.float64).T.reshape(-1) for kk in keys]))
        d = np.array(dims, dtype=np.int64)
        K = int(np.prod(d))
        out = np.zeros(K * m0 * m0 * 2)
        check(self.lib.lt_block_diagonalize(self.h, _i(d), m0, len(keys), _i(k), _d(b), _d(out)))
        z = out[0::2] + 1j * out[1::2]
        return z.reshape(K, m0, m0).transpose(0, 2, 1).copy()

    def solve_box_dense(self, H: np.ndarray, S: np.ndarray, cap: int = 4096, want_vectors: bool = False):
        """solve_box_dense (eigensolver.hpp:17-18): ascending eigenvalues, or with
        want_vectors the DenseSpectrum with S-orthonormal eigenvector columns."""
        n = H.shape[0]
        Hc = np.asfortranarray(H, dtype=np.float64)
        Sc = np.asfortranarray(S, dtype=np.float64)
        out = np.zeros(n)
        if not want_vectors:
            check(self.lib.lt_solve_box_dense(self.h, n, Hc.ctypes.data_as(_dp), Sc.ctypes.data_as(_dp), cap,
                                              _d(out)))
            return out
        vec = np.zeros(max(n * n, 1))
        check(self.lib.lt_solve_box_dense_vectors(self.h, n, Hc.ctypes.data_as(_dp), Sc.ctypes.data_as(_dp), cap,
                                                  _d(out), _d(vec)))
        return DenseSpectrum(out, vec[:n * n].reshape(n, n).T.copy())

    def pencil_eig(self, Hs: np.ndarray, Ss: np.ndarray) -> np.ndarray:
        """Batch of Hermitian-definite pencils (count, m0, m0) complex."""
        cnt, m0, _ = Hs.shape
        def pack(a):
            a = np.asarray(a, dtype=np.complex128).transpose(0, 2, 1).reshape(-1)
            o = np.empty(2 * a.size)
            o[0::2], o[1::2] = a.real, a.imag
            return o
        h, s = pack(Hs), pack(Ss)
        out = np.zeros(cnt * m0)
        check(self.lib.lt_pencil_eig(self.h, cnt, m0, _d(h), _d(s), _d(out)))
        return out.reshape(cnt, m0)

    def pencil_eigvec(self, Hs: np.ndarray, Ss: np.ndarray):
        """Batch of pencils with eigenvectors (solve_pencil with want_vectors,
        eigensolver.cpp:72-93): (eig [count, m0], vec [count, m0, m0] complex)."""
        cnt, m0, _ = Hs.shape
        h, s = _cblocks_in(Hs), _cblocks_in(Ss)
        out = np.zeros(cnt * m0)
        vec = _cvec_out(cnt * m0 * m0)
        check(self.lib.lt_pencil_eigvec(self.h, cnt, m0, _d(h), _d(s), _d(out), _d(vec)))
        return out.reshape(cnt, m0), _cblocks(vec, cnt, m0)

    def reconstruct_eigenvectors(self, spec: KPointSpectrum, cap: int = 4096) -> np.ndarray:
        """reconstruct_eigenvectors (eigensolver.cpp:164-175): the (K m0)^2 complex matrix
        whose column j m0 + m is bc_full_eigenvector(spec, j, m)."""
        if not spec.has_vectors():
            raise StructureError("reconstruct_eigenvectors: spectrum carries no eigenvectors")
        d = np.array(spec.dims, dtype=np.int64)
        N = spec.k_count() * spec.m0
        u = _cblocks_in(spec.eigenvectors)
        out = _cvec_out(N * N) if N <= cap else np.zeros(2)
        check(self.lib.lt_reconstruct_eigenvectors(self.h, _i(d), spec.m0, _d(u), cap, _d(out)))
        z = out[0::2] + 1j * out[1::2]
        return z.reshape(N, N).T.copy()

    def bc_full_eigenvector(self, spec: KPointSpectrum, j: int, m: int) -> np.ndarray:
        """bc_full_eigenvector (block_circulant.cpp:267-289): full-space vector of (j, m)."""
        if not spec.has_vectors():
            raise StructureError("bc_full_eigenvector: no eigenvectors stored")
        d = np.array(spec.dims, dtype=np.int64)
        N = spec.k_count() * spec.m0
        u = _cblocks_in(spec.eigenvectors)
        out = _cvec_out(N)
        check(self.lib.lt_bc_full_eigenvector(self.h, _i(d), spec.m0, _d(u), j, m, _d(out)))
        return out[0::2] + 1j * out[1::2]

    # ---- stages --------------------------------------------------------
    def build_sinc_quadrature(self, M: int):
        t = np.zeros(2 * M + 1)
        w = np.zeros(2 * M + 1)
        check(self.lib.lt_sinc_quadrature(self.h, M, _d(t), _d(w)))
        return t, w

    def overlap_constant(self, sys: LatticeSystem) -> int:
        c = sys.to_c()
        out = np.zeros(1, dtype=np.int64)
        check(self.lib.lt_overlap_constant(self.h, ctypes.byref(c), _i(out)))
        return int(out[0])

    def newton_master(self, ncells: int, h: float, M: int) -> np.ndarray:
        R = 2 * M + 1
        out = np.zeros(ncells * R)
        check(self.lib.lt_newton_master(self.h, ncells, h, M, _d(out)))
        return out.reshape(R, ncells).T.copy()

    def potential(self, sys: LatticeSystem, periodic: bool, margin: int):
        c = sys.to_c()
        rows = np.zeros(3, dtype=np.int64)
        tiled = np.zeros(3, dtype=np.int64)
        check(self.lib.lt_potential(self.h, ctypes.byref(c), int(periodic), margin, _i(rows), _i(tiled), None, None, 0))
        R = sys.rank_total
        total = int(rows.sum()) * R
        panels = np.zeros(total)
        w = np.zeros(R)
        check(self.lib.lt_potential(self.h, ctypes.byref(c), int(periodic), margin, _i(rows), _i(tiled), _d(panels),
                                    _d(w), total))
        out, at = [], 0
        for l in range(3):
            r = int(rows[l])
            out.append(panels[at:at + r * R].reshape(R, r).T.copy())
            at += r * R
        return out, w, tuple(bool(x) for x in tiled)

    def assembled_window_sum(self, master: np.ndarray, shifts, size: int) -> np.ndarray:
        mrows, R = master.shape
        m = np.asfortranarray(master, dtype=np.float64)
        sh = np.array(shifts, dtype=np.int64)
        out = np.zeros(size * R)
        check(self.lib.lt_assembled_window_sum(self.h, mrows, R, m.ctypes.data_as(_dp), len(sh), _i(sh), size,
                                               _d(out)))
        return out.reshape(R, size).T.copy()

    def profiles(self, sys: LatticeSystem, margin: int):
        """pwc/pwl profiles on the assembly grids: {('pwc'|'pwl', l, mu): (offset, values)}."""
        c = sys.to_c()
        grid = np.zeros(6, dtype=np.int64)
        m0 = sys.m0
        lo = np.zeros(6 * m0, dtype=np.int64)
        hi = np.zeros(6 * m0, dtype=np.int64)
        check(self.lib.lt_profiles(self.h, ctypes.byref(c), margin, _i(grid), _i(lo), _i(hi), None, 0))
        total = int(grid.sum()) * m0
        vals = np.zeros(total)
        check(self.lib.lt_profiles(self.h, ctypes.byref(c), margin, _i(grid), _i(lo), _i(hi), _d(vals), total))
        out, at = {}, 0
        for k in range(6):
            g = int(grid[k])
            for mu in range(m0):
                v = vals[at + mu * g: at + (mu + 1) * g]
                a, b = int(lo[k * m0 + mu]), int(hi[k * m0 + mu])
                out[("pwc" if k < 3 else "pwl", k % 3, mu)] = (a, v[a:b].copy())
            at += g * m0
        return out


class MultiContext:
    """Several GPUs of this process (lt_mctx): one context per device and an in-process NCCL
    communicator; solve_core shards the path across them."""

    SPLITS = {"kpoints": 0, "rankterms": 1}

    def __init__(self, devices):
        self.lib = native.lib()
        devs = (ctypes.c_int * len(devices))(*devices)
        h = ctypes.c_void_p()
        check(self.lib.lt_create_multi(devs, len(devices), ctypes.byref(h)))
        self.h = h
        self.devices = list(devices)

    def close(self):
        if self.h:
            self.lib.lt_destroy_multi(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def ndev(self) -> int:
        return int(self.lib.lt_multi_ndev(self.h))

    def solve_core(self, sys: LatticeSystem, periodic: bool, split: str = "kpoints",
                   info: Optional[np.ndarray] = None) -> np.ndarray:
        c = sys.to_c()
        out = np.zeros(sys.basis_count)
        inf = np.zeros(8, dtype=np.int64) if info is None else info
        check(self.lib.lt_solve_core_multi(self.h, ctypes.byref(c), int(periodic), self.SPLITS[split], _d(out), _i(inf)))
        return out.reshape(sys.lattice_count, sys.m0) if periodic else out


def _current_stream(device: int) -> int:
    """Raw handle of torch's current CUDA stream on `device` (the cheap accessor when present)."""
    import torch
    raw = getattr(torch._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return raw(device)
    return torch.cuda.current_stream(device).cuda_stream


class DeviceSystem:
    """A LatticeSystem resident on the device (lt_sysdev) for the bench's device-timed leg."""

    def __init__(self, ctx: Context, sys: LatticeSystem):
        self.ctx = ctx
        self.sys = sys
        c = sys.to_c()
        h = ctypes.c_void_p()
        check(ctx.lib.lt_sys_upload(ctx.h, ctypes.byref(c), ctypes.byref(h)))
        self.h = h

    @contextlib.contextmanager
    def _ordered(self, stream):
        """Order the engine's work on caller device buffers after the caller's stream (torch's
        current stream by default) and the caller's later work after the engine's."""
        if stream is None:
            import torch
            stream = torch.cuda.current_stream(self.ctx.device).cuda_stream
        check(self.ctx.lib.lt_stream_wait(self.ctx.h, ctypes.c_void_p(stream)))
        try:
            yield
        finally:
            check(self.ctx.lib.lt_stream_join(self.ctx.h, ctypes.c_void_p(stream)))

    def solve(self, periodic: bool, eig_dev_ptr: int, k_begin: int = 0, k_end: int = -1,
              info: Optional[np.ndarray] = None, stream: Optional[int] = None):
        """Solve into eig_dev_ptr, ordered after `stream` (torch's current stream by default)
        and before its later work, in one C-ABI call (lt_solve_core_dev_on)."""
        inf = np.zeros(8, dtype=np.int64) if info is None else info
        if stream is None:
            stream = _current_stream(self.ctx.device)
        check(self.ctx.lib.lt_solve_core_dev_on(self.ctx.h, self.h, int(periodic), eig_dev_ptr, k_begin, k_end,
                                                _i(inf), stream))
        return inf

    # ---- multi-GPU assembly shards (lt_core_layout / lt_assemble_core_dev / lt_spectrum_dev)
    def layout(self, periodic: bool):
        """(info, kidx): info = L0, nblocks, N_b, K, m0, R_tot, doubles per operator,
        eigenvalues per k-point; kidx [nblocks, 3] (periodic) or None."""
        info = np.zeros(8, dtype=np.int64)
        check(self.ctx.lib.lt_core_layout(self.ctx.h, self.h, int(periodic), _i(info), None))
        kidx = None
        if periodic:
            kidx = np.zeros((int(info[1]), 3), dtype=np.int64)
            check(self.ctx.lib.lt_core_layout(self.ctx.h, self.h, 1, _i(info), _i(kidx)))
        return info, kidx

    def assemble_shard(self, periodic: bool, r_begin: int, r_end: int, with_kinetic: bool, H_ptr: int, S_ptr: int,
                       stream: Optional[int] = None):
        """H shard = [0.5 Laplace] - sum_{r in [r_begin, r_end)} w_r prod_l T_l, S = Mass, into
        device buffers of layout()[0][6] doubles."""
        with self._ordered(stream):
            check(self.ctx.lib.lt_assemble_core_dev(self.ctx.h, self.h, int(periodic), int(r_begin), int(r_end),
                                                    int(bool(with_kinetic)), ctypes.c_void_p(H_ptr),
                                                    ctypes.c_void_p(S_ptr)))

    def spectrum(self, periodic: bool, H_ptr: int, S_ptr: int, eig_ptr: int, k_begin: int = 0, k_end: int = -1,
                 stream: Optional[int] = None):
        with self._ordered(stream):
            check(self.ctx.lib.lt_spectrum_dev(self.ctx.h, self.h, int(periodic), ctypes.c_void_p(H_ptr),
                                               ctypes.c_void_p(S_ptr), ctypes.c_void_p(eig_ptr), int(k_begin),
                                               int(k_end)))

    def __del__(self):
        if getattr(self, "h", None):
            try:
                self.ctx.lib.lt_sys_free(self.h)
            except Exception:
                pass
            self.h = None


_default: Optional[Context] = None


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


def assemble_box(sys: LatticeSystem, kind: str) -> Operator:
    return default_context().assemble_box(sys, kind)


def assemble_periodic(sys: LatticeSystem, kind: str) -> Operator:
    return default_context().assemble_periodic(sys, kind)


def assemble_core(sys: LatticeSystem, periodic: bool):
    return default_context().assemble_core(sys, periodic)


def combine(wa: float, a: Operator, wb: float, b: Operator) -> Operator:
    return default_context().combine(wa, a, wb, b)


def solve_periodic(H: Operator, S: Operator, want_vectors: bool = False):
    return default_context().solve_periodic(H, S, want_vectors)


def reconstruct_eigenvectors(spec: KPointSpectrum, cap: int = 4096) -> np.ndarray:
    return default_context().reconstruct_eigenvectors(spec, cap)


def bc_full_eigenvector(spec: KPointSpectrum, j: int, m: int) -> np.ndarray:
    return default_context().bc_full_eigenvector(spec, j, m)


def solve_box_dense(H: np.ndarray, S: np.ndarray, cap: int = 4096, want_vectors: bool = False):
    return default_context().solve_box_dense(H, S, cap, want_vectors)


def solve_core(sys: LatticeSystem, periodic: bool) -> np.ndarray:
    return default_context().solve_core(sys, periodic)


def spectral_bands(eig: np.ndarray):
    """spectral_bands (eigensolver.cpp:177-190): eig [K, m0] -> (bands [m0, K], band_min, band_max)."""
    eig = np.asarray(eig, dtype=np.float64)
    bands = eig.T.copy()
    return bands, bands.min(axis=1), bands.max(axis=1)


def average_energy_per_cell(sorted_eigenvalues, cells: int, n_occ: int) -> float:
    """average_energy_per_cell (eigensolver.cpp:192-198): sum of the lowest n_occ*cells / cells."""
    ev = np.asarray(sorted_eigenvalues, dtype=np.float64)
    take = n_occ * cells
    if take < 0 or take > ev.size:
        raise DimensionError("average_energy_per_cell: occupation exceeds spectrum size")
    return float(np.sum(ev[:take])) / float(cells)
