"""paper_2605_18404_b200 — B200-native JanusPipe hot path (four-phase MLIP
training step under SymFold / WaveK pipeline schedules).

The product is C++ host code (include/janus/*.hpp, csrc/*.cpp) calling
hand-written sm_100a kernels (csrc/*.cu) through the C ABI in
include/janus_cuda.h, all inside libjanus_b200.so.  This module is a thin
ctypes binding of that ABI for the tests and bench.py — plumbing, not the
product.  There is no Python or CPU fallback: if the library is missing,
import fails loudly.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

# The library does not touch the process environment.  Applications running
# many compute lanes should set CUDA_DEVICE_MAX_CONNECTIONS (one hardware work
# queue per lane, e.g. 32) before the first CUDA context exists; bench.py and
# the tests do.  janus_trainer_create warns on stderr when lanes exceed it.
# The per-rank (one process per GPU) path also needs CUDA_MODULE_LOADING=EAGER
# and a hardware queue per stream; janus_trainer_create refuses to run without.

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("JANUS_LIB") or os.path.join(_HERE, "libjanus_b200.so")  # JANUS_LIB: profiling builds only

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} not built — run `make` (or __graft_entry__.build()) first; "
                      "there is no fallback implementation")

_lib = ctypes.CDLL(LIB_PATH)

c_int, c_i64, c_u64, c_f, c_d, c_vp, c_sz = (ctypes.c_int, ctypes.c_int64, ctypes.c_uint64, ctypes.c_float,
                                              ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t)

PREC_FP32, PREC_TF32, PREC_FP32_EMU = 0, 1, 2
(PORT_ACT_IN, PORT_ACT_OUT, PORT_ADJ_IN, PORT_ADJ_OUT, PORT_TAN_IN, PORT_TAN_OUT, PORT_BADJ_IN,
 PORT_BADJ_OUT) = range(8)
METHOD_SYMFOLD, METHOD_WAVEK, METHOD_ONEF1B, METHOD_FIRST, METHOD_HANAYO = 0, 1, 2, 3, 4


class ModelDesc(ctypes.Structure):
    _fields_ = [("L", ctypes.c_int32), ("H", ctypes.c_int32), ("R", ctypes.c_int32), ("n_species", ctypes.c_int32),
                ("r_c", c_f), ("w_E", c_f), ("w_F", c_f), ("precision", ctypes.c_int32)]


class StageDesc(ctypes.Structure):
    _fields_ = [("model", ModelDesc), ("unit_begin", ctypes.c_int32), ("unit_end", ctypes.c_int32),
                ("max_atoms", ctypes.c_int32), ("max_edges", ctypes.c_int32), ("max_struct", ctypes.c_int32),
                ("n_micro_batches", ctypes.c_int32), ("n_slots", ctypes.c_int32), ("device", ctypes.c_int32),
                ("n_lanes", ctypes.c_int32), ("kernels", ctypes.c_int32)]


class HostBatch(ctypes.Structure):
    _fields_ = [("n_atoms", ctypes.c_int32), ("n_struct", ctypes.c_int32), ("n_edges", ctypes.c_int32),
                ("pos", c_vp), ("species", c_vp), ("struct_id", c_vp), ("cell", c_vp), ("E_target", c_vp),
                ("F_target", c_vp), ("row_ptr", c_vp), ("col", c_vp), ("shift", c_vp), ("rev", c_vp)]


class Opt(ctypes.Structure):
    _fields_ = [("lr", c_f), ("beta1", c_f), ("beta2", c_f), ("eps", c_f)]



def _sig(name, res, *args):
    f = getattr(_lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


_sig("janus_last_error", ctypes.c_char_p)
_sig("janus_abi_version", c_int)
_sig("janus_device_count", c_int, c_vp)
_sig("janus_param_count", c_i64, c_vp)
_sig("janus_unit_param_offset", c_i64, c_vp, c_int)
_sig("janus_num_units", c_int, c_vp)
_sig("janus_synth_params", c_int, c_vp, c_u64, c_vp)
_sig("janus_synth_cell", c_int, ctypes.c_int32, c_d, ctypes.c_int32, c_u64, c_vp, c_vp, c_vp, c_vp, c_vp)
_sig("janus_nbrlist_build", c_int, ctypes.c_int32, c_vp, c_vp, c_vp, c_d, ctypes.c_int32, c_vp, c_vp, c_vp, c_vp,
     c_vp)
_sig("janus_nbrlist_create", c_int, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, c_vp)
_sig("janus_nbrlist_destroy", c_int, c_vp)
_sig("janus_nbrlist_build_device", c_int, c_vp, ctypes.c_int32, ctypes.c_int32, c_vp, c_vp, c_vp, c_d, c_vp, c_vp,
     c_vp, c_vp, c_vp, c_vp)
_sig("janus_gars_pack", c_int, c_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, c_u64, c_vp, c_vp, c_vp)
_sig("janus_gars_greedy", c_int, c_vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, c_vp, c_vp, c_vp)
_sig("janus_gars_assign_bins", c_int, c_vp, ctypes.c_int32, ctypes.c_int32, c_vp)
_sig("janus_gars_synth_sizes", c_int, c_vp, ctypes.c_int32, c_u64, c_vp, c_vp)
_sig("janus_tune_wavek", c_int, ctypes.c_int32, ctypes.c_int32, c_vp, c_vp, ctypes.c_int32, c_vp, c_vp, c_vp,
     ctypes.c_int32, c_vp)
_sig("janus_render_timeline", c_int, c_vp, ctypes.c_int32, ctypes.c_char_p, c_vp, ctypes.c_int32, c_d, c_vp, c_i64,
     c_vp)
_sig("janus_schedule_memory", c_int, ctypes.c_char_p, c_vp, c_vp, ctypes.c_int32, c_vp, c_vp, ctypes.c_int32, c_vp)
_sig("janus_plan_stages", c_int, c_vp, ctypes.c_int32, c_vp)
_sig("janus_stage_create", c_int, c_vp, c_vp, c_vp)
_sig("janus_stage_destroy", c_int, c_vp)
_sig("janus_stage_load", c_int, c_vp, c_int, c_vp, c_vp)
for _p in ("fe", "ff", "bf", "be"):
    _sig(f"janus_stage_{_p}", c_int, c_vp, c_int, c_int, c_vp)
_sig("janus_stage_port", c_int, c_vp, c_int, c_int, c_int, c_vp, c_vp)
_sig("janus_stage_energy", c_int, c_vp, c_int, c_vp, c_vp, c_vp)
_sig("janus_stage_forces", c_int, c_vp, c_int, c_vp, c_vp, c_vp)
_sig("janus_stage_grads", c_int, c_vp, c_int, c_int, c_vp, c_vp)
_sig("janus_stage_params", c_int, c_vp, c_vp, c_vp)
_sig("janus_stage_param_count", c_i64, c_vp)
_sig("janus_stage_reduce_grads", c_int, c_vp, c_vp)
_sig("janus_stage_optimizer_step", c_int, c_vp, c_vp, c_vp)
_sig("janus_stage_memory", c_int, c_vp, c_vp, c_vp)
_sig("janus_stage_time_edge_kernel", c_int, c_vp, c_int, c_int, c_int, c_int, c_vp, c_vp, c_vp, c_vp)
_sig("janus_schedule_generate", c_int, c_int, c_int, c_int, c_int, c_vp, c_i64, c_vp)
_sig("janus_schedule_validate", c_int, ctypes.c_char_p, c_vp)


class JanusError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"janus error {code}: {msg}")
        self.code = code


def check(rc: int) -> None:
    if rc != 0:
        raise JanusError(rc, (_lib.janus_last_error() or b"").decode())


def lib():
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(c_vp)


@dataclass
class Model:
    L: int = 4
    H: int = 64
    R: int = 64
    n_species: int = 4
    r_c: float = 5.0
    w_E: float = 1.0
    w_F: float = 10.0
    precision: int = PREC_FP32
    generic: bool = False  # force the generic-width GEMM path (automatic when H or R != 64)

    def desc(self) -> ModelDesc:
        return ModelDesc(self.L, self.H, self.R, self.n_species, self.r_c, self.w_E, self.w_F, self.precision)

    @property
    def n_units(self) -> int:
        return 2 * self.L + 2

    def param_count(self) -> int:
        d = self.desc()
        return int(_lib.janus_param_count(ctypes.byref(d)))

    def unit_offset(self, u: int) -> int:
        d = self.desc()
        return int(_lib.janus_unit_param_offset(ctypes.byref(d), u))

    def synth_params(self, seed: int) -> np.ndarray:
        out = np.zeros(self.param_count(), np.float32)
        d = self.desc()
        check(_lib.janus_synth_params(ctypes.byref(d), seed, _p(out)))
        return out


class Batch:
    """One micro-batch: concatenated cubic cells + neighbour list (host arrays).

    nl="device": no host neighbour list; the load builds it on the GPU
    (janus_stage_load / janus_trainer_load with row_ptr == NULL)."""

    def __init__(self, pos, species, struct_id, cell, E_target, F_target, nl=None, r_c: float | None = None,
                 max_edges: int | None = None):
        self.pos = np.ascontiguousarray(pos, np.float64).reshape(-1, 3)
        self.species = np.ascontiguousarray(species, np.int32)
        self.struct_id = np.ascontiguousarray(struct_id, np.int32)
        self.cell = np.ascontiguousarray(cell, np.float64)
        self.E_target = np.ascontiguousarray(E_target, np.float32)
        self.F_target = np.ascontiguousarray(F_target, np.float32).reshape(-1, 3)
        if isinstance(nl, str) and nl == "device":
            nl = (None, None, None, None)
        elif nl is None:
            nl = nbrlist(self.pos, self.struct_id, self.cell, r_c, max_edges)
        self.row_ptr, self.col, self.shift, self.rev = nl

    @property
    def device_nbrlist(self) -> bool:
        return self.row_ptr is None

    @property
    def n_atoms(self):
        return self.pos.shape[0]

    @property
    def n_struct(self):
        return self.cell.shape[0]

    @property
    def n_edges(self):
        return 0 if self.row_ptr is None else int(self.col.shape[0])

    def c(self) -> HostBatch:
        q = (lambda a: None if a is None else _p(a))
        return HostBatch(self.n_atoms, self.n_struct, self.n_edges, _p(self.pos), _p(self.species),
                         _p(self.struct_id), _p(self.cell), _p(self.E_target), _p(self.F_target), q(self.row_ptr),
                         q(self.col), q(self.shift), q(self.rev))


def nbrlist(pos, struct_id, cell, r_c, max_edges=None):
    pos = np.ascontiguousarray(pos, np.float64).reshape(-1, 3)
    n = pos.shape[0]
    max_edges = max_edges or n * 400
    row_ptr = np.zeros(n + 1, np.int32)
    col = np.zeros(max_edges, np.int32)
    shift = np.zeros(3 * max_edges, np.int32)
    rev = np.zeros(max_edges, np.int32)
    ne = ctypes.c_int32(0)
    sid = np.ascontiguousarray(struct_id, np.int32)
    cl = np.ascontiguousarray(cell, np.float64)
    check(_lib.janus_nbrlist_build(n, _p(pos), _p(sid), _p(cl), r_c, max_edges, _p(row_ptr), _p(col), _p(shift),
                                   _p(rev), ctypes.byref(ne)))
    E = ne.value
    return row_ptr, col[:E].copy(), shift[:3 * E].copy(), rev[:E].copy()


def nbrlist_device(pos, struct_id, cell, r_c, max_edges=None, device: int = 0):
    """janus_nbrlist_build_device on device memory (cudart), CSR copied back."""
    pos = np.ascontiguousarray(pos, np.float64).reshape(-1, 3)
    n = pos.shape[0]
    sid = np.ascontiguousarray(struct_id, np.int32)
    cl = np.ascontiguousarray(cell, np.float64)
    max_edges = max_edges or n * 400
    rt = cudart()
    sizes = [pos.nbytes, sid.nbytes, 4 * (n + 1), 4 * max_edges, 12 * max_edges, 4 * max_edges]
    ptrs = []
    h = c_vp()
    try:
        for b in sizes:
            p = c_vp()
            if rt.cudaMalloc(ctypes.byref(p), max(b, 4)) != 0:
                raise RuntimeError("cudaMalloc failed")
            ptrs.append(p.value)
        dpos, dsid, drow, dcol, dsh, drev = ptrs
        if rt.cudaMemcpy(dpos, _p(pos), pos.nbytes, 1) or rt.cudaMemcpy(dsid, _p(sid), sid.nbytes, 1):
            raise RuntimeError("cudaMemcpy H2D failed")
        check(_lib.janus_nbrlist_create(n, len(cl), max_edges, device, ctypes.byref(h)))
        ne = ctypes.c_int32(0)
        check(_lib.janus_nbrlist_build_device(h, n, len(cl), dpos, dsid, _p(cl), r_c, drow, dcol, dsh, drev,
                                              ctypes.byref(ne), None))
        E = ne.value
        row_ptr = np.zeros(n + 1, np.int32)
        col = np.zeros(max(E, 1), np.int32)
        shift = np.zeros(max(3 * E, 1), np.int32)
        rev = np.zeros(max(E, 1), np.int32)
        for host, dev, nb in ((row_ptr, drow, 4 * (n + 1)), (col, dcol, 4 * E), (shift, dsh, 12 * E),
                              (rev, drev, 4 * E)):
            if nb and rt.cudaMemcpy(_p(host), dev, nb, 2):
                raise RuntimeError("cudaMemcpy D2H failed")
        return row_ptr, col[:E].copy(), shift[:3 * E].copy(), rev[:E].copy()
    finally:
        if h.value:
            _lib.janus_nbrlist_destroy(h)
        for p in ptrs:
            rt.cudaFree(p)


# ------------------------------------------------------------------ render
def render_timeline(recs=None, text=None, t=None, svg=False, quantum=1.0) -> str:
    """ASCII / SVG timeline of executor records ([n][5]: device, phase, mb, start, end)
    or of a schedule text replayed under phase times t = (FE, FF, BE, BF)."""
    r = None if recs is None else np.ascontiguousarray(recs, np.float64)
    tt = None if t is None else np.ascontiguousarray(t, np.float64)
    args = (None if r is None else _p(r), 0 if r is None else r.shape[0], None if text is None else text.encode(),
            None if tt is None else _p(tt), 1 if svg else 0, quantum)
    n = c_i64()
    check(_lib.janus_render_timeline(*args, None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value + 1)
    check(_lib.janus_render_timeline(*args, buf, n.value + 1, ctypes.byref(n)))
    return buf.value.decode()


# ------------------------------------------------------------------ tuner
def tune_wavek(P: int, n_mb: int, t, m_gpu: float, m_reserve: float, m_static: float, fe_bytes: float,
               ff_bytes: float, stage0_mult: float = 1.0, divisors_only: bool = True):
    """janus_tune_wavek: (k_star, tuned, rows of {k, makespan, bubble_ratio, peak_max, feasible})."""
    tt = np.ascontiguousarray(t, np.float64)
    mem = np.array([m_gpu, m_reserve, m_static, fe_bytes, ff_bytes, stage0_mult], np.float64)
    ks, tu, n = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
    table = np.zeros((max(n_mb, 1), 5))
    check(_lib.janus_tune_wavek(P, n_mb, _p(tt), _p(mem), 1 if divisors_only else 0, ctypes.byref(ks),
                                ctypes.byref(tu), _p(table), table.shape[0], ctypes.byref(n)))
    rows = [dict(k=int(r[0]), makespan=float(r[1]), bubble_ratio=float(r[2]), peak_max=float(r[3]),
                 feasible=bool(r[4])) for r in table[:n.value]]
    return ks.value, bool(tu.value), rows


def plan_stages(model: "Model", P: int) -> np.ndarray:
    """Unit ranges [P][2] of the trainer's stage partition (no device needed)."""
    out = np.zeros((P, 2), np.int32)
    d = model.desc()
    check(_lib.janus_plan_stages(ctypes.byref(d), P, _p(out)))
    return out


def schedule_memory(text: str, t, static_bytes, fe_bytes: float, ff_bytes: float, stage0_mult: float = 1.0,
                    replicate: bool = True):
    """Lifetime-rule peak bytes per device of a schedule replayed under t (janus_schedule_memory)."""
    tt = np.ascontiguousarray(t, np.float64)
    st = np.ascontiguousarray(np.atleast_1d(static_bytes), np.float64)
    act = np.array([fe_bytes, ff_bytes, stage0_mult, 1.0 if replicate else 0.0], np.float64)
    out = np.zeros(256)
    n = ctypes.c_int32()
    check(_lib.janus_schedule_memory(text.encode(), _p(tt), _p(st), len(st), _p(act), _p(out), 256, ctypes.byref(n)))
    return out[:n.value].copy()


# ------------------------------------------------------------------ GARS
def gars_pack(atoms, n_mb: int, d_gp: int = 1, seed: int = 0, greedy: bool = False):
    """janus_gars_pack (or the greedy sequential baseline): list of
    (graph ids in micro-batch order, tag) per micro-batch; tag 0 comm_free, 1 dist."""
    a = np.ascontiguousarray(atoms, np.int32)
    order = np.zeros(len(a), np.int32)
    ptr = np.zeros(n_mb + 1, np.int32)
    tags = np.zeros(n_mb, np.int32)
    if greedy:
        check(_lib.janus_gars_greedy(_p(a), len(a), n_mb, d_gp, _p(order), _p(ptr), _p(tags)))
    else:
        check(_lib.janus_gars_pack(_p(a), len(a), n_mb, d_gp, seed, _p(order), _p(ptr), _p(tags)))
    return [(order[ptr[j]:ptr[j + 1]].tolist(), int(tags[j])) for j in range(n_mb)]


def gars_assign_bins(sizes, d_gp: int):
    a = np.ascontiguousarray(sizes, np.int32)
    out = np.zeros(len(a), np.int32)
    check(_lib.janus_gars_assign_bins(_p(a), len(a), d_gp, _p(out)))
    return out.tolist()


def gars_synth_sizes(n: int, seed: int, stats=None):
    a = np.zeros(n, np.int32)
    e = np.zeros(n, np.int64)
    st = None if stats is None else np.ascontiguousarray(stats, np.float64)
    check(_lib.janus_gars_synth_sizes(None if st is None else _p(st), n, seed, _p(a), _p(e)))
    return a, e


def synth_cell(n_atoms: int, rho: float, n_species: int, seed: int):
    pos = np.zeros((n_atoms, 3))
    sp = np.zeros(n_atoms, np.int32)
    cell = ctypes.c_double(0)
    Et = np.zeros(1, np.float32)
    Ft = np.zeros((n_atoms, 3), np.float32)
    check(_lib.janus_synth_cell(n_atoms, rho, n_species, seed, _p(pos), _p(sp), ctypes.byref(cell), _p(Et), _p(Ft)))
    return pos, sp, cell.value, float(Et[0]), Ft


def synth_batch(model: Model, atoms_per_cell, rho: float, seed: int, device_nl: bool = False) -> Batch:
    """A micro-batch of one or more synthetic cells (sizes in atoms_per_cell).
    device_nl: leave the neighbour list to the GPU load (no host CSR)."""
    if isinstance(atoms_per_cell, int):
        atoms_per_cell = [atoms_per_cell]
    P, S, SID, C, E, F = [], [], [], [], [], []
    for s, n in enumerate(atoms_per_cell):
        pos, sp, L, Et, Ft = synth_cell(n, rho, model.n_species, seed * 1000003 + s)
        P.append(pos); S.append(sp); SID.append(np.full(n, s, np.int32)); C.append(L); E.append(Et); F.append(Ft)
    return Batch(np.concatenate(P), np.concatenate(S), np.concatenate(SID), np.array(C), np.array(E),
                 np.concatenate(F), r_c=model.r_c, nl="device" if device_nl else None)


class Stage:
    """A pipeline stage on one GPU (units [u0, u1))."""

    def __init__(self, model: Model, params_all: np.ndarray, u0: int, u1: int, max_atoms: int, max_edges: int,
                 max_struct: int = 8, n_mb: int = 1, n_slots: int = 1, device: int = 0):
        self.model = model
        self.u0, self.u1 = u0, u1
        o0, o1 = model.unit_offset(u0), model.unit_offset(u1)
        self.param_slice = slice(o0, o1)
        sl = np.ascontiguousarray(params_all[o0:o1], np.float32)
        self.desc = StageDesc(model.desc(), u0, u1, max_atoms, max_edges, max_struct, n_mb, n_slots, device, 1,
                              1 if model.generic else 0)
        h = c_vp()
        check(_lib.janus_stage_create(ctypes.byref(self.desc), _p(sl), ctypes.byref(h)))
        self.h = h

    def close(self):
        if self.h:
            check(_lib.janus_stage_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load(self, mb: int, batch: Batch, stream=None):
        hb = batch.c()
        check(_lib.janus_stage_load(self.h, mb, ctypes.byref(hb), stream))

    def fe(self, mb, slot=None, stream=None):
        check(_lib.janus_stage_fe(self.h, mb, mb if slot is None else slot, stream))

    def ff(self, mb, slot=None, stream=None):
        check(_lib.janus_stage_ff(self.h, mb, mb if slot is None else slot, stream))

    def bf(self, mb, slot=None, stream=None):
        check(_lib.janus_stage_bf(self.h, mb, mb if slot is None else slot, stream))

    def be(self, mb, slot=None, stream=None):
        check(_lib.janus_stage_be(self.h, mb, mb if slot is None else slot, stream))

    def port(self, mb, slot, port):
        ptr, nb = c_vp(), c_sz()
        check(_lib.janus_stage_port(self.h, mb, slot, port, ctypes.byref(ptr), ctypes.byref(nb)))
        return ptr.value, nb.value

    def energy(self, mb, n_struct):
        E = np.zeros(n_struct, np.float32)
        l = np.zeros(1, np.float32)
        check(_lib.janus_stage_energy(self.h, mb, _p(E), _p(l), None))
        return E, float(l[0])

    def forces(self, mb, n_atoms):
        F = np.zeros((n_atoms, 3), np.float32)
        l = np.zeros(1, np.float32)
        check(_lib.janus_stage_forces(self.h, mb, _p(F), _p(l), None))
        return F, float(l[0])

    def param_count(self):
        return int(_lib.janus_stage_param_count(self.h))

    def grads(self, which=0, mb=-1):
        out = np.zeros(self.param_count(), np.float32)
        check(_lib.janus_stage_grads(self.h, which, mb, _p(out), None))
        return out

    def params(self):
        out = np.zeros(self.param_count(), np.float32)
        check(_lib.janus_stage_params(self.h, _p(out), None))
        return out

    def grad_buffer(self) -> np.ndarray:
        """The reduced gradient OS applied (after any pair / data-parallel all-reduce)."""
        ptr, n = c_vp(), c_i64()
        check(_lib.janus_stage_grad_buffer(self.h, ctypes.byref(ptr), ctypes.byref(n)))
        out = np.zeros(n.value, np.float32)
        rt = cudart()
        assert rt.cudaDeviceSynchronize() == 0
        assert rt.cudaMemcpy(out.ctypes.data, ptr.value, out.nbytes, 2) == 0
        return out

    def reduce_grads(self, stream=None):
        check(_lib.janus_stage_reduce_grads(self.h, stream))

    def optimizer_step(self, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, stream=None):
        o = Opt(lr, beta1, beta2, eps)
        check(_lib.janus_stage_optimizer_step(self.h, ctypes.byref(o), stream))

    def time_edge_kernel(self, which: int, mb: int = 0, slot: int | None = None, iters: int = 20):
        """Mean launch time (ms), edges and algorithmic FLOPs of one msg edge kernel."""
        ms, ne, fl = c_f(), c_i64(), c_d()
        check(_lib.janus_stage_time_edge_kernel(self.h, which, mb, mb if slot is None else slot, iters, None,
                                                ctypes.byref(ms), ctypes.byref(ne), ctypes.byref(fl)))
        return ms.value, ne.value, fl.value

    def memory(self):
        a, b = c_i64(), c_i64()
        check(_lib.janus_stage_memory(self.h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value


def schedule_text(method: int, P: int, n_mb: int, k: int = 1) -> str:
    n = c_i64()
    check(_lib.janus_schedule_generate(method, P, n_mb, k, None, 0, ctypes.byref(n)))
    buf = ctypes.create_string_buffer(n.value + 1)
    check(_lib.janus_schedule_generate(method, P, n_mb, k, buf, n.value + 1, ctypes.byref(n)))
    return buf.value.decode()


def validate_schedule(text: str) -> int:
    n = ctypes.c_int32()
    check(_lib.janus_schedule_validate(text.encode(), ctypes.byref(n)))
    return n.value


_sig("janus_schedule_replay", c_int, ctypes.c_char_p, c_vp, c_vp, c_vp)


def schedule_replay(text: str, t_fe: float, t_ff: float, t_be: float, t_bf: float):
    """Replay a schedule under phase times -> (makespan, bubble ratio)."""
    t = np.array([t_fe, t_ff, t_be, t_bf], np.float64)
    ms, br = c_d(), c_d()
    check(_lib.janus_schedule_replay(text.encode(), _p(t), ctypes.byref(ms), ctypes.byref(br)))
    return ms.value, br.value


_sig("janus_schedule_check_rendezvous", c_int, ctypes.c_char_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
     ctypes.c_int32, c_vp, c_vp, c_vp, ctypes.c_char_p, c_i64)


def check_rendezvous(text: str, onef1b: bool = False, lanes: int = 1, dp: int = 1, shared_streams: bool = False):
    """Blocking-rendezvous simulation of the multi-process issue program ->
    (ok, completed ops, total ops, stuck stream heads)."""
    ok, done, tot = ctypes.c_int32(), c_i64(), c_i64()
    buf = ctypes.create_string_buffer(4096)
    check(_lib.janus_schedule_check_rendezvous(text.encode(), 1 if onef1b else 0, lanes, dp, 1 if shared_streams else 0,
                                               ctypes.byref(ok), ctypes.byref(done), ctypes.byref(tot), buf, 4096))
    return bool(ok.value), done.value, tot.value, buf.value.decode()


_sig("janus_schedule_slot_pool", c_int, ctypes.c_char_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
     ctypes.c_int32, c_vp, ctypes.c_int32, c_vp)


def slot_pool(text: str, onef1b: bool = False, local: bool = True, unfolded: bool = False, lanes: int = 1):
    """Activation slots per device the executor allocates for a schedule
    (include/janus/slots.hpp): the live micro-batches of its largest pool."""
    out = np.zeros(64, np.int32)
    n = ctypes.c_int32()
    check(_lib.janus_schedule_slot_pool(text.encode(), 1 if onef1b else 0, 1 if local else 0, 1 if unfolded else 0,
                                        lanes, _p(out), 64, ctypes.byref(n)))
    return out[:n.value].tolist()


def device_count() -> int:
    n = c_int()
    check(_lib.janus_device_count(ctypes.byref(n)))
    return n.value


# ----------------------------------------------------------- cudart helpers
_cudart = None


def cudart():
    """libcudart for D2D copies in single-GPU multi-stage tests (fake transport)."""
    global _cudart
    if _cudart is None:
        for name in ("libcudart.so", "libcudart.so.12"):
            try:
                _cudart = ctypes.CDLL(name)
                break
            except OSError:
                continue
        if _cudart is None:
            raise ImportError("libcudart not found")
        _cudart.cudaMemcpy.argtypes = [c_vp, c_vp, c_sz, c_int]
        _cudart.cudaMemcpy.restype = c_int
        _cudart.cudaMalloc.argtypes = [c_vp, c_sz]
        _cudart.cudaMalloc.restype = c_int
        _cudart.cudaFree.argtypes = [c_vp]
        _cudart.cudaFree.restype = c_int
        _cudart.cudaDeviceSynchronize.restype = c_int
    return _cudart


def d2d(dst: int, src: int, nbytes: int) -> None:
    rc = cudart().cudaMemcpy(dst, src, nbytes, 3)  # cudaMemcpyDeviceToDevice
    if rc != 0:
        raise RuntimeError(f"cudaMemcpy failed: {rc}")


# ------------------------------------------------------------------ trainer
class StepStats(ctypes.Structure):
    _fields_ = [("makespan_ms", c_d), ("bubble_ratio", c_d), ("busy_ms", c_d * 64), ("p2p_bytes", c_i64),
                ("kernel_launches", c_i64), ("peak_bytes", c_i64 * 64), ("loss", c_d), ("act_bytes", c_i64 * 64),
                ("act_slots", ctypes.c_int32 * 64)]


class ExecDesc(ctypes.Structure):
    _fields_ = [("n_stages", ctypes.c_int32), ("method", ctypes.c_int32), ("wavek_k", ctypes.c_int32),
                ("n_micro_batches", ctypes.c_int32), ("local_stages", ctypes.c_int32), ("use_graphs", ctypes.c_int32),
                ("dp_degree", ctypes.c_int32), ("record_timeline", ctypes.c_int32), ("lanes", ctypes.c_int32),
                ("unfolded_slots", ctypes.c_int32), ("phase_us", ctypes.c_double * 4)]


_sig("janus_trainer_create", c_int, c_vp, c_vp, c_vp, c_vp, c_int, c_vp)
_sig("janus_trainer_destroy", c_int, c_vp)
_sig("janus_trainer_load", c_int, c_vp, c_int, c_vp)
_sig("janus_trainer_step", c_int, c_vp, c_vp, c_vp)
_sig("janus_trainer_step_async", c_int, c_vp, c_vp)
_sig("janus_trainer_wait", c_int, c_vp, c_vp)
_sig("janus_trainer_timeline", c_int, c_vp, c_vp, ctypes.c_int32, c_vp)
_sig("janus_trainer_stage", c_int, c_vp, c_int, c_int, c_vp)
_sig("janus_trainer_schedule_text", c_int, c_vp, c_vp, c_i64, c_vp)
_sig("janus_trainer_plan", c_int, c_vp, c_vp)
_sig("janus_nccl_unique_id", c_int, c_vp)
_sig("janus_comm_init_nccl", c_int, c_vp, c_int, c_int, c_int, c_vp)
_sig("janus_comm_init_ipc", c_int, ctypes.c_char_p, c_int, c_int, c_int, c_vp)
_sig("janus_comm_init_threads", c_int, ctypes.c_char_p, c_int, c_int, c_int, c_vp)
_sig("janus_comm_destroy", c_int, c_vp)


class _StageView(Stage):
    """Non-owning view of a stage held by a trainer."""

    def __init__(self, model, handle, u0, u1):  # no super().__init__: the trainer owns it
        self.model, self.h, self.u0, self.u1 = model, handle, u0, u1

    def close(self):
        self.h = None


class Comm:
    """Per-rank communicator (one per process; rank r holds pipeline device
    r % P of replica r // P): NCCL, or the same-GPU IPC transport (Comm.ipc)."""

    def __init__(self, uid: bytes | None, nranks: int, rank: int, device: int, ipc_dir: str | None = None,
                 threads: bool = False):
        h = c_vp()
        if ipc_dir is not None:
            init = _lib.janus_comm_init_threads if threads else _lib.janus_comm_init_ipc
            check(init(ipc_dir.encode(), nranks, rank, device, ctypes.byref(h)))
        else:
            buf = ctypes.create_string_buffer(uid, 128)
            check(_lib.janus_comm_init_nccl(buf, nranks, rank, device, ctypes.byref(h)))
        self.h = h

    @classmethod
    def ipc(cls, rendezvous_dir: str, nranks: int, rank: int, device: int = 0) -> "Comm":
        """N processes on ONE GPU with NCCL's blocking-rendezvous semantics
        (CUDA IPC staging + stream memory operations; csrc/transport.hpp)."""
        return cls(None, nranks, rank, device, ipc_dir=rendezvous_dir)

    @classmethod
    def threads(cls, rendezvous_dir: str, nranks: int, rank: int, device: int = 0) -> "Comm":
        """N ranks as threads of THIS process on one GPU, same protocol (one CUDA
        context, so the ranks' kernels run concurrently)."""
        return cls(None, nranks, rank, device, ipc_dir=rendezvous_dir, threads=True)

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        check(_lib.janus_nccl_unique_id(buf))
        return buf.raw

    def close(self):
        if self.h:
            check(_lib.janus_comm_destroy(self.h))
            self.h = None


class Trainer:
    """janus_trainer: executes a SymFold / WaveK / 1F1B-2nd schedule (C++)."""

    def __init__(self, model: Model, params: np.ndarray, P: int, method: int, n_mb: int, k: int = 1,
                 max_atoms: int = 256, max_edges: int = 256 * 120, max_struct: int = 8, local: bool = True,
                 graphs: bool = False, timeline: bool = False, dp: int = 1, comm: "Comm | None" = None,
                 rank: int = 0, device: int = 0, lanes: int = 1, unfolded: bool = False, phase_us=None):
        """unfolded=True: one activation slot per micro-batch instead of the
        schedule-sized pool (include/janus/slots.hpp), for memory A/B studies.
        phase_us = measured (FE, FF, BE, BF) times for WaveK's cost model."""
        self.model, self.P, self.n_mb = model, P, n_mb
        self.ed = ExecDesc(P, method, k, n_mb, 1 if local else 0, 1 if graphs else 0, dp, 1 if timeline else 0,
                           lanes, 1 if unfolded else 0, (ctypes.c_double * 4)(*(phase_us or (0, 0, 0, 0))))
        self.sd = StageDesc(model.desc(), 0, model.n_units, max_atoms, max_edges, max_struct, n_mb, n_mb, device,
                            lanes, 1 if model.generic else 0)
        p = np.ascontiguousarray(params, np.float32)
        h = c_vp()
        check(_lib.janus_trainer_create(ctypes.byref(self.ed), ctypes.byref(self.sd), _p(p),
                                        comm.h if comm else None, rank, ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            check(_lib.janus_trainer_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def load(self, mb: int, batch: Batch):
        hb = batch.c()
        check(_lib.janus_trainer_load(self.h, mb, ctypes.byref(hb)))

    def load_many(self, batches, mbs=None):
        """LM of several micro-batches; device-LM batches share one GPU build."""
        mbs = list(range(len(batches))) if mbs is None else list(mbs)
        arr = (HostBatch * len(batches))(*[b.c() for b in batches])
        ids = np.ascontiguousarray(mbs, np.int32)
        check(_lib.janus_trainer_load_many(self.h, len(batches), _p(ids), arr))

    def step(self, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8) -> StepStats:
        o = Opt(lr, beta1, beta2, eps)
        s = StepStats()
        check(_lib.janus_trainer_step(self.h, ctypes.byref(o), ctypes.byref(s)))
        return s

    def step_async(self, lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8) -> None:
        """Issue a step and return; loads issued before wait() queue behind it."""
        o = Opt(lr, beta1, beta2, eps)
        check(_lib.janus_trainer_step_async(self.h, ctypes.byref(o)))

    def wait(self) -> StepStats:
        s = StepStats()
        check(_lib.janus_trainer_wait(self.h, ctypes.byref(s)))
        return s

    def timeline(self):
        n = ctypes.c_int32()
        check(_lib.janus_trainer_timeline(self.h, None, 0, ctypes.byref(n)))
        out = np.zeros((max(n.value, 1), 5))
        check(_lib.janus_trainer_timeline(self.h, _p(out), n.value, ctypes.byref(n)))
        return out[:n.value]

    def plan(self):
        out = np.zeros((self.P, 2), np.int32)
        check(_lib.janus_trainer_plan(self.h, _p(out)))
        return out

    def stage(self, block: int, force_replica: bool = False) -> Stage:
        h = c_vp()
        check(_lib.janus_trainer_stage(self.h, block, 1 if force_replica else 0, ctypes.byref(h)))
        u0, u1 = self.plan()[block]
        return _StageView(self.model, h, int(u0), int(u1))

    def schedule_text(self) -> str:
        n = c_i64()
        check(_lib.janus_trainer_schedule_text(self.h, None, 0, ctypes.byref(n)))
        buf = ctypes.create_string_buffer(n.value + 1)
        check(_lib.janus_trainer_schedule_text(self.h, buf, n.value + 1, ctypes.byref(n)))
        return buf.value.decode()

    def params(self) -> np.ndarray:
        """Full parameter vector gathered from the energy copies."""
        return np.concatenate([self.stage(b).params() for b in range(self.P)])

    def grads(self, which=0) -> np.ndarray:
        """Per-micro-batch-ledger sums (energy copies; 1F1B force replicas hold the rest)."""
        return np.concatenate([self.stage(b).grads(which, -1) for b in range(self.P)])
