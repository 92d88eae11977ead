"""ctypes front-end of the C oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
legs may import this module; it is the checker, never the product path.
Every function restates a reference symbol (file:line cited in
``gsde_oracle.c``).  Graph/field inputs are anything exposing the
reference's packed attributes (``edge_length``, ``v_off``, ... and
``field.packed()``) -- both ``graphsde`` and ``paper_2512_02175_b200`` do.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liborc.so")
_lib = None

P = C.c_void_p
i64, u64, f64, i32 = C.c_int64, C.c_uint64, C.c_double, C.c_int32


class _Graph(C.Structure):
    _fields_ = [
        ("n_edges", i64), ("n_vertices", i64),
        ("edge_len", P), ("edge_init", P), ("edge_term", P),
        ("v_off", P), ("v_edges", P), ("v_orient", P), ("v_cumw", P),
        ("dkind", P), ("dcoef", P), ("tab_off", P), ("tab_x", P), ("tab_mu", P), ("sigma", P),
    ]


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
            os.path.join(_HERE, "gsde_oracle.c")
        ):
            build()
        L = C.CDLL(_LIB_PATH)
        L.orc_raw64.restype = u64
        L.orc_raw64.argtypes = [u64, u64, u64]
        L.orc_u64_to_uniform.restype = f64
        L.orc_u64_to_uniform.argtypes = [u64]
        L.orc_u64_to_normal.restype = f64
        L.orc_u64_to_normal.argtypes = [u64]
        L.orc_norm_ppf.restype = f64
        L.orc_norm_ppf.argtypes = [f64]
        L.orc_solve_first_passage_s.restype = f64
        L.orc_solve_first_passage_s.argtypes = [f64, f64, f64]
        L.orc_philox4x32_10.argtypes = [P, P, P]
        L.orc_step.argtypes = [C.POINTER(_Graph), i32, i64, f64, f64, u64, u64, u64, i64, f64,
                               P, P, P, P, P, P]
        L.orc_step_rows.argtypes = [C.POINTER(_Graph), i32, i64] + [P] * 15
        L.orc_trace.argtypes = [C.POINTER(_Graph), i32, u64, i64, i64, i64, f64, i32, i64, f64,
                                f64, i64, f64, P, P, P, P, P, P, i32]
        L.orc_ensemble.argtypes = [C.POINTER(_Graph), i32, u64, i64, i64, i64, f64, i32, i64,
                                   f64, f64, i64, f64, P, P, P, P, P, P, i32]
        L.orc_vertex_trials.argtypes = [C.POINTER(_Graph), i32, u64, i64, i64, f64, i64, f64,
                                        i64, P, P, P, P, i32]
        L.orc_histogram.argtypes = [i64, P, P, P, P, P, P]
        L.orc_max_threads.restype = C.c_int
        L.orc_ensemble_occupation.argtypes = [C.POINTER(_Graph), i32, u64, i64, i64, i64, f64,
                                              i32, i64, f64, f64, i64, f64, P, P, P, i64, i64,
                                              P, i32]
        L.orc_fill_draws.argtypes = [u64, u64, i64, u64, i64, P, P, i32]
        L.orc_fill_draws_rows.argtypes = [P, P, P, i64, i64, P, P]
        L.orc_fvm_steps.restype = i64
        L.orc_fvm_steps.argtypes = [P, i64, i64, f64, P, i64, P, P, P, P, P, i64, P, P, P, P, P,
                                    f64]
        _lib = L
    return _lib


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


class OracleGraph:
    """Packed graph + field held in C-compatible arrays."""

    def __init__(self, graph, field):
        kind, coef, tab_off, tab_x, tab_mu, sigma = field.packed()
        self.arrays = dict(
            edge_len=np.ascontiguousarray(graph.edge_length, np.float64),
            edge_init=np.ascontiguousarray(graph.edge_init, np.int64),
            edge_term=np.ascontiguousarray(graph.edge_term, np.int64),
            v_off=np.ascontiguousarray(graph.v_off, np.int64),
            v_edges=np.ascontiguousarray(graph.v_edges, np.int64),
            v_orient=np.ascontiguousarray(graph.v_orient, np.int8),
            v_cumw=np.ascontiguousarray(graph.v_cumw, np.float64),
            dkind=np.ascontiguousarray(kind, np.int8),
            dcoef=np.ascontiguousarray(coef, np.float64),
            tab_off=np.ascontiguousarray(tab_off, np.int64),
            tab_x=np.ascontiguousarray(tab_x if len(tab_x) else np.zeros(1), np.float64),
            tab_mu=np.ascontiguousarray(tab_mu if len(tab_mu) else np.zeros(1), np.float64),
            sigma=np.ascontiguousarray(sigma, np.float64),
        )
        self.is_star = bool(graph.is_star)
        self.n_edges = int(graph.edge_length.shape[0])
        self.n_vertices = int(graph.v_off.shape[0] - 1)
        self.edge_length = self.arrays["edge_len"]
        self.c = _Graph(self.n_edges, self.n_vertices, *[_ptr(self.arrays[k]) for k in (
            "edge_len", "edge_init", "edge_term", "v_off", "v_edges", "v_orient", "v_cumw",
            "dkind", "dcoef", "tab_off", "tab_x", "tab_mu", "sigma")])


def philox4x32_10(ctr, key):
    c = np.asarray(ctr, np.uint32)
    k = np.asarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_ptr(c), _ptr(k), _ptr(out))
    return [int(v) for v in out]


def raw64(seed, stream, index):
    return int(lib().orc_raw64(seed, stream, index))


def uniform01(seed, stream, index):
    return lib().orc_u64_to_uniform(lib().orc_raw64(seed, stream, index))


def normal(seed, stream, index):
    return lib().orc_u64_to_normal(lib().orc_raw64(seed, stream, index))


def norm_ppf(p):
    return lib().orc_norm_ppf(p)


def solve_first_passage_s(a, b, c):
    return lib().orc_solve_first_passage_s(a, b, c)


def step(og: OracleGraph, edge, x, dt, seed, pid, k, cap=100, reflect_len=0.0):
    """One macro step (``em_step_star`` / ``em_step_general`` semantics)."""
    e = np.zeros(1, np.int64); xo = np.zeros(1); M = np.zeros(1, np.int64)
    tr = np.zeros(1, np.int32); ko = np.zeros(1, np.uint64)
    lib().orc_step(C.byref(og.c), int(og.is_star), edge, x, dt, seed, pid, k, cap, reflect_len,
                   _ptr(e), _ptr(xo), _ptr(M), _ptr(tr), _ptr(ko), None)
    return int(e[0]), float(xo[0]), int(M[0]), bool(tr[0]), int(ko[0])


def step_rows(og: OracleGraph, edge, x, dt, seed, pid, k, cap, reflect_len):
    """Per-row single steps (arrays of equal length n) -> dict of outputs incl.
    each step's decision ``margin`` (smallest relative distance of a
    continuous decision from its threshold; see orc_step_out)."""
    n = len(edge)
    a = lambda v, t: np.ascontiguousarray(np.broadcast_to(np.asarray(v, t), (n,)))
    ins = [a(edge, np.int64), a(x, np.float64), a(dt, np.float64), a(seed, np.uint64),
           a(pid, np.uint64), a(k, np.uint64), a(cap, np.int64), a(reflect_len, np.float64)]
    out = dict(edge=np.zeros(n, np.int64), x=np.zeros(n), M=np.zeros(n, np.int64),
               trunc=np.zeros(n, np.int32), k=np.zeros(n, np.uint64), margin=np.zeros(n))
    lib().orc_step_rows(C.byref(og.c), int(og.is_star), n, *[_ptr(v) for v in ins],
                        *[_ptr(out[q]) for q in ("edge", "x", "M", "trunc", "k", "margin")])
    return out


def trace(og: OracleGraph, seed, n, n_steps, dt, init=(0, 0, 0.0, 0.0), cap=100,
          reflect_len=0.0, pid_offset=0, threads=0):
    """Whole reference trajectories recorded after every step: arrays
    ``[n, n_steps]`` of edge, x, M, trunc, next draw index k and margin."""
    init_kind, init_edge, init_x, init_xmax = init
    out = dict(edge=np.zeros((n, n_steps), np.int64), x=np.zeros((n, n_steps)),
               M=np.zeros((n, n_steps), np.int64), trunc=np.zeros((n, n_steps), np.int32),
               k=np.zeros((n, n_steps), np.uint64), margin=np.zeros((n, n_steps)))
    lib().orc_trace(C.byref(og.c), int(og.is_star), seed, n, pid_offset, n_steps, dt, init_kind,
                    init_edge, init_x, init_xmax, cap, reflect_len,
                    *[_ptr(out[q]) for q in ("edge", "x", "M", "trunc", "k", "margin")], threads)
    return out


CHUNK = 4096


def ensemble(og: OracleGraph, seed, n, n_steps, dt, init=(0, 0, 0.0, 0.0), cap=100,
             reflect_len=0.0, pid_offset=0, threads=0):
    """``run_ensemble`` kernel semantics; returns dict of reference-dtype arrays."""
    init_kind, init_edge, init_x, init_xmax = init
    n_chunks = max(1, -(-n // CHUNK))
    out = dict(
        edges=np.zeros(n, np.int64), positions=np.zeros(n), crossings=np.zeros(n, np.int64),
        crossing_events=np.zeros(n, np.int64), truncs=np.zeros(n, np.int64),
    )
    mh = np.zeros((n_chunks, cap + 1), np.int64)
    lib().orc_ensemble(C.byref(og.c), int(og.is_star), seed, n, pid_offset, n_steps, dt,
                       init_kind, init_edge, init_x, init_xmax, cap, reflect_len,
                       _ptr(out["edges"]), _ptr(out["positions"]), _ptr(out["crossings"]),
                       _ptr(out["crossing_events"]), _ptr(out["truncs"]), _ptr(mh), threads)
    out["m_histogram"] = mh.sum(axis=0)
    return out


def vertex_trials(og: OracleGraph, seed, n, dt, start_edge=0, start_x=0.0, cap=100,
                  trial_offset=0, threads=0):
    out = dict(M=np.zeros(n, np.int64), exit_edges=np.zeros(n, np.int64),
               exit_positions=np.zeros(n), truncated=np.zeros(n, np.int64))
    lib().orc_vertex_trials(C.byref(og.c), int(og.is_star), seed, n, trial_offset, dt,
                            start_edge, start_x, cap, _ptr(out["M"]), _ptr(out["exit_edges"]),
                            _ptr(out["exit_positions"]), _ptr(out["truncated"]), threads)
    return out


def histogram(edges, positions, offsets, counts, dx):
    edges = np.ascontiguousarray(edges, np.int64)
    positions = np.ascontiguousarray(positions, np.float64)
    offsets = np.ascontiguousarray(offsets, np.int64)
    counts = np.ascontiguousarray(counts, np.int64)
    dx = np.ascontiguousarray(dx, np.float64)
    h = np.zeros(int(counts.sum()), np.int64)
    lib().orc_histogram(edges.shape[0], _ptr(edges), _ptr(positions), _ptr(offsets),
                        _ptr(counts), _ptr(dx), _ptr(h))
    return h


def max_threads():
    return int(lib().orc_max_threads())


def fill_draws(seed, n, K, pid0=0, k0=0, threads=0):
    """Reference-stream draws ``[n, K]`` (raw uint64, normals float64) for INJECT."""
    raw = np.zeros((n, K), np.uint64)
    nrm = np.zeros((n, K), np.float64)
    lib().orc_fill_draws(seed, pid0, n, k0, K, _ptr(raw), _ptr(nrm), threads)
    return raw, nrm


def fill_draws_rows(seeds, pids, k0s, K):
    seeds = np.ascontiguousarray(seeds, np.uint64)
    pids = np.ascontiguousarray(pids, np.uint64)
    k0s = np.ascontiguousarray(k0s, np.uint64)
    n = seeds.shape[0]
    raw = np.zeros((n, K), np.uint64)
    nrm = np.zeros((n, K), np.float64)
    lib().orc_fill_draws_rows(_ptr(seeds), _ptr(pids), _ptr(k0s), n, K, _ptr(raw), _ptr(nrm))
    return raw, nrm


def ensemble_occupation(og: OracleGraph, seed, n, n_steps, dt, offsets, counts, dx, every=1,
                        start=0, init=(0, 0, 0.0, 0.0), cap=100, reflect_len=0.0, pid_offset=0,
                        threads=0):
    """Time-integrated occupation histogram (samples after every ``every``-th
    step beyond ``start``), reference streams."""
    offsets = np.ascontiguousarray(offsets, np.int64)
    counts = np.ascontiguousarray(counts, np.int64)
    dx = np.ascontiguousarray(dx, np.float64)
    occ = np.zeros(int(counts.sum()), np.int64)
    init_kind, init_edge, init_x, init_xmax = init
    lib().orc_ensemble_occupation(C.byref(og.c), int(og.is_star), seed, n, pid_offset, n_steps,
                                  dt, init_kind, init_edge, init_x, init_xmax, cap, reflect_len,
                                  _ptr(offsets), _ptr(counts), _ptr(dx), every, start, _ptr(occ),
                                  threads)
    return occ


def fvm_steps(rho, n_steps, dt, packed, neg_floor=-1e-10):
    """_fvm_step_loop restated in C: advances ``rho`` (copied) over the
    ``_pack_static`` tuple; returns (rho, 1-based negative step or 0)."""
    i8, f8 = np.int64, np.float64
    kinds = (i8, f8, f8, f8, i8, i8, i8, f8, f8, f8, f8)
    (offs, dx_edge, D_edge, face_mu, face_off, v_off, v_cells, v_b, v_dx, v_sp, v_D) = [
        np.ascontiguousarray(a, dtype=k) for a, k in zip(packed, kinds)]
    if face_mu.size == 0:
        face_mu = np.zeros(1)
    rho = np.array(rho, dtype=np.float64, copy=True)
    neg = lib().orc_fvm_steps(_ptr(rho), rho.shape[0], int(n_steps), float(dt), _ptr(offs),
                              dx_edge.shape[0], _ptr(dx_edge), _ptr(D_edge), _ptr(face_mu),
                              _ptr(face_off), _ptr(v_off), v_off.shape[0] - 1, _ptr(v_cells),
                              _ptr(v_b), _ptr(v_dx), _ptr(v_sp), _ptr(v_D), float(neg_floor))
    return rho, int(neg)
