"""oracle/oracle.py — TEST INFRASTRUCTURE: ctypes front-end to the fp64 CPU
oracle (oracle/_ref/libmlip_oracle.so, built from oracle/mlip_oracle.c by
oracle/Makefile).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this module.  See oracle/mlip_oracle.h for scope and for how
the oracle is pinned (PyTorch fp64 autograd goldens, finite differences,
staged == unstaged, Eq. (2) ledger).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_ref", "libmlip_oracle.so")
_lib = None


class _Model(ctypes.Structure):
    _fields_ = [("L", ctypes.c_int), ("H", ctypes.c_int), ("R", ctypes.c_int), ("n_species", ctypes.c_int),
                ("r_c", ctypes.c_double), ("w_E", ctypes.c_double), ("w_F", ctypes.c_double)]


class _Batch(ctypes.Structure):
    _fields_ = [("n_atoms", ctypes.c_int), ("n_struct", ctypes.c_int),
                ("pos", ctypes.c_void_p), ("species", ctypes.c_void_p), ("struct_id", ctypes.c_void_p),
                ("cell", ctypes.c_void_p), ("E_target", ctypes.c_void_p), ("F_target", ctypes.c_void_p)]


def build() -> None:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.mo_param_count.restype = ctypes.c_int64
        L.mo_unit_param_offset.restype = ctypes.c_int64
        L.mo_unit_param_count.restype = ctypes.c_int64
        L.mo_build_nbrlist.restype = ctypes.c_int64
        _lib = L
    return _lib


@dataclass
class Model:
    L: int = 4
    H: int = 64
    R: int = 64
    n_species: int = 4
    r_c: float = 5.0
    w_E: float = 1.0
    w_F: float = 10.0

    def c(self):
        return _Model(self.L, self.H, self.R, self.n_species, self.r_c, self.w_E, self.w_F)

    @property
    def n_units(self) -> int:
        return 2 * self.L + 2

    def param_count(self) -> int:
        m = self.c()
        return int(lib().mo_param_count(ctypes.byref(m)))

    def unit_param_range(self, u: int):
        m = self.c()
        off = int(lib().mo_unit_param_offset(ctypes.byref(m), u))
        n = int(lib().mo_unit_param_count(ctypes.byref(m), u))
        return off, n


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


class Batch:
    """Concatenated periodic cubic cells (atoms of a structure contiguous)."""

    def __init__(self, pos, species, struct_id, cell, E_target, F_target):
        self.pos = np.ascontiguousarray(pos, dtype=np.float64).reshape(-1, 3)
        self.species = np.ascontiguousarray(species, dtype=np.int32)
        self.struct_id = np.ascontiguousarray(struct_id, dtype=np.int32)
        self.cell = np.ascontiguousarray(cell, dtype=np.float64)
        self.E_target = np.ascontiguousarray(E_target, dtype=np.float64)
        self.F_target = np.ascontiguousarray(F_target, dtype=np.float64).reshape(-1, 3)

    @property
    def n_atoms(self):
        return self.pos.shape[0]

    @property
    def n_struct(self):
        return self.cell.shape[0]

    def c(self):
        return _Batch(self.n_atoms, self.n_struct, _p(self.pos), _p(self.species), _p(self.struct_id),
                      _p(self.cell), _p(self.E_target), _p(self.F_target))


@dataclass
class NbrList:
    row_ptr: np.ndarray
    col: np.ndarray
    shift: np.ndarray
    rev: np.ndarray

    @property
    def n_edges(self):
        return int(self.col.shape[0])


def build_nbrlist(model: Model, batch: Batch, max_edges: int | None = None) -> NbrList:
    if max_edges is None:
        max_edges = batch.n_atoms * 400
    row_ptr = np.zeros(batch.n_atoms + 1, np.int32)
    col = np.zeros(max_edges, np.int32)
    shift = np.zeros(3 * max_edges, np.int32)
    rev = np.zeros(max_edges, np.int32)
    m, b = model.c(), batch.c()
    E = lib().mo_build_nbrlist(ctypes.byref(m), ctypes.byref(b), ctypes.c_int64(max_edges), _p(row_ptr),
                               _p(col), _p(shift), _p(rev))
    if E < 0:
        raise ValueError("neighbour list overflow")
    return NbrList(row_ptr, col[:E].copy(), shift[:3 * E].reshape(E, 3).copy(), rev[:E].copy())


@dataclass
class StepResult:
    E: np.ndarray
    F: np.ndarray
    loss: float
    grad: np.ndarray
    grad1: np.ndarray
    grad2: np.ndarray
    trace: np.ndarray | None


def step(model: Model, batch: Batch, nl: NbrList, params: np.ndarray, want_trace: bool = False) -> StepResult:
    params = np.ascontiguousarray(params, dtype=np.float64)
    NP = model.param_count()
    assert params.shape == (NP,)
    E = np.zeros(batch.n_struct)
    F = np.zeros((batch.n_atoms, 3))
    loss = np.zeros(1)
    g, g1, g2 = np.zeros(NP), np.zeros(NP), np.zeros(NP)
    trace = np.zeros((model.n_units, 8, batch.n_atoms, model.H)) if want_trace else None
    m, b = model.c(), batch.c()
    sh = np.ascontiguousarray(nl.shift.reshape(-1), dtype=np.int32)
    rc = lib().mo_step(ctypes.byref(m), ctypes.byref(b), ctypes.c_int64(nl.n_edges), _p(nl.row_ptr), _p(nl.col),
                       _p(sh), _p(nl.rev), _p(params), _p(E), _p(F), _p(loss), _p(g), _p(g1), _p(g2),
                       _p(trace) if trace is not None else None)
    assert rc == 0
    return StepResult(E, F, float(loss[0]), g, g1, g2, trace)


def energy(model: Model, batch: Batch, nl: NbrList, params: np.ndarray) -> np.ndarray:
    params = np.ascontiguousarray(params, dtype=np.float64)
    E = np.zeros(batch.n_struct)
    m, b = model.c(), batch.c()
    sh = np.ascontiguousarray(nl.shift.reshape(-1), dtype=np.int32)
    lib().mo_energy(ctypes.byref(m), ctypes.byref(b), ctypes.c_int64(nl.n_edges), _p(nl.row_ptr), _p(nl.col),
                    _p(sh), _p(params), _p(E))
    return E


def adam(p, m1, m2, g, lr, beta1, beta2, eps, step_no):
    for a in (p, m1, m2):
        assert a.dtype == np.float64 and a.flags.c_contiguous
    g = np.ascontiguousarray(g, dtype=np.float64)
    lib().mo_adam(ctypes.c_int64(p.size), _p(p), _p(m1), _p(m2), _p(g), ctypes.c_double(lr),
                  ctypes.c_double(beta1), ctypes.c_double(beta2), ctypes.c_double(eps), ctypes.c_int(step_no))


def synth_params(model: Model, seed: int) -> np.ndarray:
    """Seeded parameters, bit-identical to the product's janus_synth_params."""
    out = np.zeros(model.param_count(), np.float32)
    m = model.c()
    L = lib()
    L.mo_synth_params.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p]
    L.mo_synth_params(ctypes.byref(m), ctypes.c_uint64(seed), _p(out))
    return out


def synth_cell(n: int, rho: float, n_species: int, seed: int):
    """(pos [n,3] f64, species [n] i32, box length, E_target f32, F_target [n,3] f32),
    bit-identical to the product's janus_synth_cell."""
    pos = np.zeros((n, 3), np.float64)
    sp = np.zeros(n, np.int32)
    Et = np.zeros(1, np.float32)
    Ft = np.zeros((n, 3), np.float32)
    L = lib()
    L.mo_synth_cell.restype = ctypes.c_double
    L.mo_synth_cell.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_int, ctypes.c_uint64, ctypes.c_void_p,
                                ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
    box = L.mo_synth_cell(n, rho, n_species, ctypes.c_uint64(seed), _p(pos), _p(sp), _p(Et), _p(Ft))
    if box < 0:
        raise ValueError("synth_cell: bad arguments")
    return pos, sp, box, float(Et[0]), Ft


def synth_batch(model: Model, atoms_per_cell, rho: float, seed: int) -> Batch:
    """The product's synth_batch (paper_2605_18404_b200.synth_batch) restated:
    cell s of the batch is seeded with seed * 1000003 + s."""
    if isinstance(atoms_per_cell, int):
        atoms_per_cell = [atoms_per_cell]
    P, S, SID, C, E, F = [], [], [], [], [], []
    for s, n in enumerate(atoms_per_cell):
        pos, sp, box, Et, Ft = synth_cell(n, rho, model.n_species, seed * 1000003 + s)
        P.append(pos); S.append(sp); SID.append(np.full(n, s, np.int32)); C.append(box); E.append(Et)
        F.append(Ft)
    return Batch(np.concatenate(P), np.concatenate(S), np.concatenate(SID), np.array(C),
                 np.array(E, np.float32).astype(np.float64), np.concatenate(F).astype(np.float64))
