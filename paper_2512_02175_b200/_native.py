"""ctypes binding of ``libgsde.so`` (the C ABI declared in ``include/gsde.h``).

The library is built in-tree (``__graft_entry__.build()`` / ``make -C
paper_2512_02175_b200/csrc``).  There is no fallback: if the library is
missing or no CUDA device is usable, simulation calls raise
:class:`NativeUnavailable`.  Device memory and streams come from PyTorch
(plumbing only); every kernel is ours.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# GSDE_LIB_PATH: an alternative build of the same library (A/B kernel experiments)
LIB_PATH = os.environ.get("GSDE_LIB_PATH") or os.path.join(_HERE, "libgsde.so")

GSDE_STREAM_NATIVE = 0
GSDE_STREAM_REFERENCE = 1
GSDE_STREAM_INJECT = 2
GSDE_PREC_F32 = 0
GSDE_PREC_F64 = 1
GSDE_PREC_NATIVE = 2  # INJECT into the production FP32 kernel (ensembles)
GSDE_INIT_POINT = 0
GSDE_INIT_PER_EDGE_UNIFORM = 1
GSDE_INIT_STATE = 2

_P = C.c_void_p
_i64, _u64, _f64, _i32 = C.c_int64, C.c_uint64, C.c_double, C.c_int32


class NativeUnavailable(RuntimeError):
    """libgsde.so is missing or no sm_100 CUDA device is usable."""


class GsdeError(RuntimeError):
    def __init__(self, code: int, message: str):
        self.code = code
        super().__init__(f"gsde error {code}: {message}")


class GraphDesc(C.Structure):
    _fields_ = [
        ("n_edges", _i64), ("n_vertices", _i64), ("n_tab", _i64),
        ("edge_length", _P), ("edge_init", _P), ("edge_term", _P),
        ("v_off", _P), ("v_edges", _P), ("v_orient", _P), ("v_cumw", _P), ("v_weights", _P),
        ("dkind", _P), ("dcoef", _P), ("tab_off", _P), ("tab_x", _P), ("tab_mu", _P),
        ("sigma", _P), ("is_star", _i32),
    ]


class Run(C.Structure):
    _fields_ = [
        ("seed", _u64), ("n_particles", _i64), ("pid_offset", _i64), ("n_steps", _i64),
        ("dt", _f64), ("init_kind", _i32), ("init_edge", _i64), ("init_x", _f64),
        ("init_xmax", _f64), ("cap", _i32), ("reflect_len", _f64), ("stream", _i32),
        ("precision", _i32), ("inj_raw", _P), ("inj_normal", _P), ("inj_stride", _i64),
        ("state_edge", _P), ("state_x", _P), ("state_counter", _P),
    ]


class Out(C.Structure):
    _fields_ = [
        ("edge", _P), ("crossings", _P), ("events", _P), ("truncs", _P), ("x", _P),
        ("m_hist", _P), ("totals", _P), ("edge_counts", _P), ("hist", _P),
        ("hist_offsets", _P), ("hist_counts", _P), ("hist_dx", _P), ("hist_n_cells", _i64),
        ("occ", _P), ("occ_every", _i64), ("occ_start", _i64), ("counter", _P),
        ("progress", _P), ("progress_base", _i64), ("progress_shift", _i32),
    ]


class Trials(C.Structure):
    _fields_ = [
        ("seed", _u64), ("n_trials", _i64), ("trial_offset", _i64), ("dt", _f64),
        ("start_edge", _i64), ("start_x", _f64), ("cap", _i32), ("stream", _i32),
        ("precision", _i32), ("inj_raw", _P), ("inj_normal", _P), ("inj_stride", _i64),
    ]


class TrialsOut(C.Structure):
    _fields_ = [
        ("M", _P), ("edge", _P), ("trunc", _P), ("x", _P), ("exit_counts", _P),
        ("m_hist", _P), ("totals", _P),
    ]


class StepArgs(C.Structure):
    _fields_ = [
        ("n", _i64), ("dt", _f64), ("cap", _i32), ("reflect_len", _f64), ("stream", _i32),
        ("precision", _i32), ("seed", _P), ("pid", _P), ("inj_raw", _P), ("inj_normal", _P),
        ("inj_stride", _i64),
    ]


#: Every symbol include/gsde.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "gsde_graph_create", "gsde_graph_destroy", "gsde_graph_device_bytes", "gsde_ensemble",
    "gsde_vertex_trials", "gsde_step_batch", "gsde_histogram", "gsde_raw64", "gsde_uniform01",
    "gsde_normal", "gsde_solve_first_passage_s", "gsde_launch_count", "gsde_abi_version",
    "gsde_last_error", "gsde_parse_graph_text", "gsde_parsed_sizes", "gsde_parsed_export",
    "gsde_parsed_free", "gsde_fvm_run", "gsde_u64_to_uniform", "gsde_u64_to_normal",
    "gsde_norm_ppf", "gsde_stream_wait_geq32",
)

_lib = None
_lock = threading.Lock()


def lib():
    """Load libgsde.so (no GPU needed to load it)."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not os.path.exists(LIB_PATH):
                    raise NativeUnavailable(
                        f"{LIB_PATH} not built; run __graft_entry__.build() or "
                        "`make -C paper_2512_02175_b200/csrc`"
                    )
                L = C.CDLL(LIB_PATH)
                L.gsde_graph_create.argtypes = [C.POINTER(GraphDesc), C.c_int, C.POINTER(_P)]
                L.gsde_graph_destroy.argtypes = [_P]
                L.gsde_graph_device_bytes.argtypes = [_P]
                L.gsde_graph_device_bytes.restype = _i64
                L.gsde_ensemble.argtypes = [_P, C.POINTER(Run), C.POINTER(Out), _P]
                L.gsde_vertex_trials.argtypes = [_P, C.POINTER(Trials), C.POINTER(TrialsOut), _P]
                L.gsde_stream_wait_geq32.argtypes = [_P, _P, C.c_uint32]
                L.gsde_step_batch.argtypes = [_P, C.POINTER(StepArgs), _P, _P, _P, _P, _P, _P]
                L.gsde_histogram.argtypes = [_i64, _P, _P, _P, _P, _P, _i64, _P, _P]
                L.gsde_fvm_run.argtypes = [_P, _P, _P, _i64, _f64, _f64, _P, _P, _P]
                L.gsde_raw64.argtypes = [_u64, _u64, _u64]
                L.gsde_raw64.restype = _u64
                for name in ("gsde_uniform01", "gsde_normal"):
                    getattr(L, name).argtypes = [_u64, _u64, _u64]
                    getattr(L, name).restype = _f64
                for name in ("gsde_u64_to_uniform", "gsde_u64_to_normal"):
                    getattr(L, name).argtypes = [_u64]
                    getattr(L, name).restype = _f64
                L.gsde_norm_ppf.argtypes = [_f64]
                L.gsde_norm_ppf.restype = _f64
                L.gsde_solve_first_passage_s.argtypes = [_f64, _f64, _f64]
                L.gsde_solve_first_passage_s.restype = _f64
                L.gsde_parse_graph_text.argtypes = [C.c_char_p, _i64, C.POINTER(_P)]
                L.gsde_parsed_sizes.argtypes = [_P, _P]
                L.gsde_parsed_sizes.restype = None
                L.gsde_parsed_export.argtypes = [_P] * 18
                L.gsde_parsed_export.restype = None
                L.gsde_parsed_free.argtypes = [_P]
                L.gsde_parsed_free.restype = None
                L.gsde_launch_count.restype = _i64
                L.gsde_last_error.restype = C.c_char_p
                assert L.gsde_abi_version() == 3, "libgsde ABI mismatch"
                _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().gsde_last_error()
        raise GsdeError(rc, msg.decode() if msg else "unknown")


def torch_cuda(device=None):
    """Return (torch, device index) or raise NativeUnavailable."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the simulator runs on the GPU only")
    if device is None:
        device = torch.cuda.current_device()
    return torch, int(device)


def ptr(t):
    return None if t is None else t.data_ptr()


def cur_stream(device: int):
    import torch

    return torch.cuda.current_stream(device).cuda_stream


class DeviceGraph:
    """A graph + coefficient field resident on one GPU (opaque library handle)."""

    def __init__(self, graph, field, device=None):
        torch, device = torch_cuda(device)
        L = lib()
        kind, coef, tab_off, tab_x, tab_mu, sigma = field.packed()
        self._keep = arrs = dict(
            edge_length=np.ascontiguousarray(graph.edge_length, np.float64),
            edge_init=np.ascontiguousarray(graph.edge_init, np.int64),
            edge_term=np.ascontiguousarray(graph.edge_term, np.int64),
            v_off=np.ascontiguousarray(graph.v_off, np.int64),
            v_edges=np.ascontiguousarray(graph.v_edges, np.int64),
            v_orient=np.ascontiguousarray(graph.v_orient, np.int8),
            v_cumw=np.ascontiguousarray(graph.v_cumw, np.float64),
            v_weights=np.ascontiguousarray(graph.v_weights, np.float64),
            dkind=np.ascontiguousarray(kind, np.int8),
            dcoef=np.ascontiguousarray(coef, np.float64),
            tab_off=np.ascontiguousarray(tab_off, np.int64),
            tab_x=np.ascontiguousarray(tab_x if len(tab_x) else np.zeros(1), np.float64),
            tab_mu=np.ascontiguousarray(tab_mu if len(tab_mu) else np.zeros(1), np.float64),
            sigma=np.ascontiguousarray(sigma, np.float64),
        )
        d = GraphDesc()
        d.n_edges = graph.n_edges
        d.n_vertices = graph.n_vertices
        d.n_tab = int(len(tab_x))
        for k, a in arrs.items():
            setattr(d, k, a.ctypes.data)
        d.is_star = int(graph.is_star)
        h = _P()
        check(L.gsde_graph_create(C.byref(d), device, C.byref(h)))
        self.handle = h
        self.device = device
        self.n_edges = graph.n_edges
        self.is_star = bool(graph.is_star)
        self._keep = None

    @property
    def device_bytes(self) -> int:
        return int(lib().gsde_graph_device_bytes(self.handle))

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and _lib is not None:
            try:
                _lib.gsde_graph_destroy(h)
            except Exception:
                pass
            self.handle = None


def device_graph(graph, field, device=None) -> DeviceGraph:
    """Cached upload of (graph, field) to ``device``: one entry per device --
    the most recent field (a sweep that builds a new field per point frees
    the previous point's device arena instead of keeping one per field)."""
    _, device = torch_cuda(device)
    cache = graph._device
    key = ("dg", device)
    hit = cache.get(key)
    if hit is not None and hit[0] is field:
        return hit[1]
    cache.pop(key, None)  # drop the old handle first: its arena returns to the pool
    dg = DeviceGraph(graph, field, device)
    cache[key] = (field, dg)
    return dg


def launch_count() -> int:
    return int(lib().gsde_launch_count())
