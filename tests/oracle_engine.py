"""Oracle-backed stand-in for the engine's device-buffer interface (TEST INFRASTRUCTURE).

paper_1408_3839_b200/dist.py drives any context whose upload(sys) returns an object with the
DeviceSystem methods — solve / layout / assemble_shard / spectrum, writing through buffer
pointers — so the real multi-rank functions (solve_core_distributed, solve_core_sharded,
_gather_k) run on CPU tensors under gloo with this stand-in in place of the CUDA engine.
Buffer layouts follow include/latham_b200.h (lt_core_layout): periodic operators as
[nblocks][m0*m0] generating blocks in kidx order, each block column-major; eigenvalues
[K][m0] k-lexicographic, ascending per k.
"""
from __future__ import annotations

import ctypes

import numpy as np


def _view(ptr: int, n: int) -> np.ndarray:
    return np.ctypeslib.as_array(ctypes.cast(ctypes.c_void_p(ptr), ctypes.POINTER(ctypes.c_double)), shape=(n,))


class OracleContext:
    def __init__(self):
        from oracle.binding import oracle
        import torch
        self.o = oracle()
        self.torch_device = torch.device("cpu")

    def upload(self, sys):
        return OracleSystem(self, sys)


class OracleSystem:
    def __init__(self, ctx: OracleContext, sys):
        self.o = ctx.o
        self.sys = sys
        self._core = {}

    def _assembled(self, periodic):
        if periodic not in self._core:
            self._core[periodic] = self.o.assemble_core(self.sys, periodic)
        return self._core[periodic]

    # ---- lt_solve_core_dev
    def solve(self, periodic, eig_ptr, k_begin=0, k_end=-1, info=None, stream=None):
        H, S = self._assembled(periodic)
        if periodic:
            ev = self.o.solve_periodic_ops(H, S)
            K = ev.shape[0]
            k_end = K if k_end < 0 or k_end > K else k_end
            out = _view(eig_ptr, ev.size).reshape(ev.shape)
            out[k_begin:k_end] = ev[k_begin:k_end]
        else:
            ev = self.o.solve_box_dense(H.dense, S.dense)
            _view(eig_ptr, ev.size)[:] = ev
        if info is not None:
            info[0] = H.L0
        return info

    # ---- lt_core_layout
    def layout(self, periodic):
        H, _ = self._assembled(periodic)
        s = self.sys
        m0 = s.m0
        nuc = self.o.assemble(s, periodic, "nuclear")
        Rtot = nuc.coefficient_rank
        self.o.free(nuc)
        if periodic:
            nblk = H.kidx.shape[0]
            info = np.array([H.L0, nblk, s.basis_count, s.lattice_count, m0, Rtot, nblk * m0 * m0, m0], dtype=np.int64)
            return info, H.kidx.copy()
        nb = s.basis_count
        return np.array([H.L0, 0, nb, s.lattice_count, m0, Rtot, nb * nb, nb], dtype=np.int64), None

    # ---- lt_assemble_core_dev: H shard = [0.5 Laplace] - sum_{r in [r0, r1)} w_r prod_l T_l
    def assemble_shard(self, periodic, r0, r1, with_kinetic, H_ptr, S_ptr, stream=None):
        if not periodic:
            raise NotImplementedError("oracle stand-in: rank-term shards of box systems")
        s, o = self.sys, self.o
        H, S = self._assembled(True)
        keys = [tuple(int(x) for x in k) for k in H.kidx]
        lap = o.assemble(s, True, "laplace")
        nuc = o.assemble(s, True, "nuclear")
        ld = lap.gen_dict()
        terms = o.separable_terms(nuc)  # one term per nuclear rank term, weight in level 0
        r1 = len(terms) if r1 < 0 else min(r1, len(terms))
        m0 = s.m0
        Hout = _view(H_ptr, len(keys) * m0 * m0).reshape(len(keys), m0, m0)
        Sout = _view(S_ptr, len(keys) * m0 * m0).reshape(len(keys), m0, m0)
        sd = S.gen_dict()
        for i, k in enumerate(keys):
            acc = np.zeros((m0, m0))
            for t in range(r0, r1):
                acc += terms[t][0][k[0]] * terms[t][1][k[1]] * terms[t][2][k[2]]
            blk = (0.5 * ld[k] if with_kinetic else 0.0) - acc
            Hout[i] = blk.T  # [row, col] -> column-major block
            Sout[i] = sd[k].T
        o.free(lap)
        o.free(nuc)

    # ---- lt_spectrum_dev
    def spectrum(self, periodic, H_ptr, S_ptr, eig_ptr, k_begin=0, k_end=-1, stream=None):
        if not periodic:
            raise NotImplementedError("oracle stand-in: dense spectrum from buffers")
        s = self.sys
        info, kidx = self.layout(True)
        m0, nblk = s.m0, int(info[1])
        keys = [tuple(int(x) for x in k) for k in kidx]
        Hb = _view(H_ptr, nblk * m0 * m0).reshape(nblk, m0, m0)
        Sb = _view(S_ptr, nblk * m0 * m0).reshape(nblk, m0, m0)
        Hg = {k: Hb[i].T.copy() for i, k in enumerate(keys)}
        Sg = {k: Sb[i].T.copy() for i, k in enumerate(keys)}
        ev = self.o.solve_periodic(s.L, m0, Hg, Sg)
        K = ev.shape[0]
        k_end = K if k_end < 0 or k_end > K else k_end
        out = _view(eig_ptr, ev.size).reshape(ev.shape)
        out[k_begin:k_end] = ev[k_begin:k_end]
