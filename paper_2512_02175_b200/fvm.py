"""Finite-volume Fokker-Planck baseline (reference ``graphsde/fvm.py``), stepped on the GPU.

The density on each edge evolves under ``d(rho)/dt = -dF/dx`` with
``F = mu rho - D d(rho)/dx``, ``D = sigma^2 / 2``: upwind drift and central
diffusion on interior faces, explicit Euler in time, and at every vertex of
degree >= 2 a pairwise, jump-weight-normalised mass exchange between the
vertex-adjacent cells (``fvm.py:1-27`` states the scheme).

``fvm_run`` packs the static per-face / per-slot coefficients exactly like
``_pack_static`` (``fvm.py:343-382``), uploads them once and runs every step
in ONE persistent cooperative kernel (``csrc/gsde_fvm.cu`` via
``gsde_fvm_run``) that reproduces ``_fvm_step_loop``'s floating-point
operation order, so the density is bit-identical to the reference's.
The diagnostic helpers (``fvm_interior_fluxes``, ``fvm_vertex_fluxes``,
``stability_limit``) are host-side numpy restatements.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _native
from .coefficients import CoefficientField, ConstantDrift, LinearDrift, eval_diffusion, eval_drift
from .graph import AT_INIT, MetricGraph
from .grids import EdgeGrid

#: Relative negative-density threshold that flags a blown-up solution (``fvm.py:41``).
_NEGATIVE_TOL = 1e-10


class UnstableTimestep(RuntimeError):
    pass


class NegativeDensity(RuntimeError):
    pass


class ZeroJumpWeightAtVertex(ValueError):
    pass


@dataclass
class FvmState:
    """Flat per-cell densities (probability per unit length) on a grid (``fvm.py:59-89``)."""

    grid: EdgeGrid
    rho: np.ndarray
    t: float = 0.0

    @classmethod
    def uniform(cls, grid: EdgeGrid, mass: float = 1.0) -> "FvmState":
        total_len = float(grid.lengths.sum())
        return cls(grid=grid, rho=np.full(grid.n_cells, mass / total_len, dtype=np.float64), t=0.0)

    @classmethod
    def from_function(cls, grid: EdgeGrid, f) -> "FvmState":
        """Sample ``f(edge, x_center)`` on cell centers (no normalization)."""
        rho = np.empty(grid.n_cells, dtype=np.float64)
        for e in range(grid.n_edges):
            rho[grid.edge_slice(e)] = [f(e, float(x)) for x in grid.centers(e)]
        return cls(grid=grid, rho=rho, t=0.0)

    def mass(self) -> float:
        return float(np.dot(self.rho, self.grid.cell_widths()))

    def edge_density(self, e: int) -> np.ndarray:
        return self.rho[self.grid.edge_slice(e)]

    def copy(self) -> "FvmState":
        return FvmState(grid=self.grid, rho=self.rho.copy(), t=self.t)


@dataclass(frozen=True)
class FvmResult:
    state: FvmState
    max_cfl: float
    n_steps: int


def _drift_at(field: CoefficientField, e: int, xs: np.ndarray) -> np.ndarray:
    """``eval_drift`` on an array of positions (same IEEE results as the scalar calls)."""
    spec = field.drift[e]
    if isinstance(spec, ConstantDrift):
        return np.full(xs.shape, spec.c, dtype=np.float64)
    if isinstance(spec, LinearDrift):
        return spec.c * xs
    return np.interp(xs, spec.xs, spec.mus).astype(np.float64)


def _drift_pairs(field: CoefficientField, edges: np.ndarray, xs: np.ndarray) -> np.ndarray:
    """``eval_drift(field, edges[k], xs[k])`` for every k, vectorised: the same
    IEEE operation per element as the scalar calls (constant: c; linear: c * x;
    tabulated: np.interp on the edge's samples)."""
    edges = np.asarray(edges, dtype=np.int64)
    xs = np.asarray(xs, dtype=np.float64)
    kind, coef, _, _, _, _ = field.packed()
    k = np.asarray(kind)[edges]
    c = np.asarray(coef, dtype=np.float64)[edges]
    out = np.where(k == 1, c * xs, c)
    tab = np.flatnonzero(k == 2)
    if tab.size:
        for e in np.unique(edges[tab]).tolist():
            sel = tab[edges[tab] == e]
            spec = field.drift[e]
            out[sel] = np.interp(xs[sel], spec.xs, spec.mus)
    return out


def _face_drift(field: CoefficientField, e: int, grid: EdgeGrid) -> np.ndarray:
    """Drift on the interior faces of edge e (``fvm.py:99-103``)."""
    return _drift_at(field, e, np.arange(1, int(grid.counts[e])) * grid.dx[e])


def fvm_interior_fluxes(state: FvmState, field: CoefficientField, grid: EdgeGrid):
    """Per-edge interior face fluxes ``mu rho_upwind - D (rho_r - rho_l) / dx``
    (``fvm.py:106-123``)."""
    out = []
    for e in range(grid.n_edges):
        rho = state.edge_density(e)
        dx = float(grid.dx[e])
        mu = _face_drift(field, e, grid)
        D = 0.5 * eval_diffusion(field, e, 0.0) ** 2
        left, right = rho[:-1], rho[1:]
        out.append(np.where(mu > 0.0, mu * left, mu * right) + (-D * (right - left) / dx))
    return out


def _vertex_slots(graph: MetricGraph, field: CoefficientField, grid: EdgeGrid, v: int):
    """``(cells, b, dx, speed_in, D)`` over the incident slots of v (``fvm.py:126-152``)."""
    inc = graph.incidence[v]
    offs = grid.offsets
    deg = inc.degree
    cells = np.empty(deg, dtype=np.int64)
    dxs, speed_in, D_v = np.empty(deg), np.empty(deg), np.empty(deg)
    for i, (eid, orient) in enumerate(zip(inc.edges, inc.orientations)):
        eid = int(eid)
        if orient == AT_INIT:
            cells[i], x_v = offs[eid], 0.0
        else:
            cells[i], x_v = offs[eid + 1] - 1, float(grid.lengths[eid])
        mu = eval_drift(field, eid, x_v)
        speed_in[i] = max(0.0, -mu if orient == AT_INIT else mu)
        D_v[i] = 0.5 * eval_diffusion(field, eid, x_v) ** 2
        dxs[i] = grid.dx[eid]
    return cells, inc.jump_weights.astype(np.float64), dxs, speed_in, D_v


def _zero_weight(v):
    return ZeroJumpWeightAtVertex(
        f"vertex {v}: the rho/b normalization needs strictly positive jump weights")


def fvm_vertex_fluxes(state: FvmState, field: CoefficientField, graph: MetricGraph,
                      grid: EdgeGrid, v: int):
    """``(net, drift_pairs, diff_pairs)`` of the exchange at v (``fvm.py:155-206``)."""
    inc = graph.incidence[v]
    deg = inc.degree
    drift_pairs = np.zeros((deg, deg))
    diff_pairs = np.zeros((deg, deg))
    if deg < 2:
        return np.zeros(deg), drift_pairs, diff_pairs
    if np.any(inc.jump_weights <= 0.0):
        raise _zero_weight(v)
    cells, b, dxs, speed_in, D_v = _vertex_slots(graph, field, grid, v)
    rho = state.rho[cells]
    conc = rho / b
    for i in range(deg):
        others = 1.0 - b[i]
        if speed_in[i] <= 0.0 or others <= 0.0:
            continue
        total = speed_in[i] * rho[i]
        for j in range(deg):
            if j != i:
                drift_pairs[i, j] = total * b[j] / others
    for i in range(deg):
        for j in range(i + 1, deg):
            dpair = 0.5 * (D_v[i] + D_v[j])
            dxh = 2.0 * dxs[i] * dxs[j] / (dxs[i] + dxs[j])
            g = dpair * (conc[i] - conc[j]) / dxh
            if g >= 0.0:
                diff_pairs[i, j] = g * b[j]
            else:
                diff_pairs[j, i] = -g * b[i]
    flows = drift_pairs + diff_pairs
    return flows.sum(axis=0) - flows.sum(axis=1), drift_pairs, diff_pairs


@dataclass(frozen=True)
class _Packed:
    """``_pack_static`` (``fvm.py:343-382``) + the GPU's ownership split."""

    offs: np.ndarray
    dx_edge: np.ndarray
    D_edge: np.ndarray
    face_mu: np.ndarray
    face_off: np.ndarray
    v_off: np.ndarray
    v_cells: np.ndarray
    v_b: np.ndarray
    v_dx: np.ndarray
    v_speed_in: np.ndarray
    v_D: np.ndarray
    cell_edge: np.ndarray
    owned: np.ndarray
    vpar: np.ndarray
    vser: np.ndarray
    slot_vertex: np.ndarray
    pslot: np.ndarray
    # two-phase vertex exchange (see _term_layout): destination ranges per pslot
    # entry, per-row write positions, and the number of terms
    tstart: np.ndarray
    rstart: np.ndarray
    rpos: np.ndarray
    n_terms: int
    # per-cell records of the GPU stepper: drift on the left / right interior
    # face, D and dx of the cell's edge, flags (1 left face, 2 right face, 4 owned)
    cell_mu_l: np.ndarray
    cell_mu_r: np.ndarray
    cell_D: np.ndarray
    cell_dx: np.ndarray
    cell_flags: np.ndarray

    def reference_tuple(self):
        return (self.offs, self.dx_edge, self.D_edge, self.face_mu, self.face_off, self.v_off,
                self.v_cells, self.v_b, self.v_dx, self.v_speed_in, self.v_D)


_PACK_MEMO: list = []  # [(graph, field, grid, packed)]: the last packing, by identity


def _pack(graph: MetricGraph, field: CoefficientField, grid: EdgeGrid) -> _Packed:
    """``_pack_static`` restated (``fvm.py:343-382``), vectorised; the last result
    is reused for the same (frozen) graph / field / grid objects -- ``fvm_run``
    needs it twice (the CFL check and the device upload)."""
    if _PACK_MEMO and all(a is b for a, b in zip(_PACK_MEMO[0][:3], (graph, field, grid))):
        return _PACK_MEMO[0][3]
    packed = _pack_uncached(graph, field, grid)
    _PACK_MEMO[:] = [(graph, field, grid, packed)]
    return packed


def _pack_uncached(graph: MetricGraph, field: CoefficientField, grid: EdgeGrid) -> _Packed:
    E = grid.n_edges
    counts = np.asarray(grid.counts, np.int64)
    offs = grid.offsets
    dx = np.asarray(grid.dx, np.float64)
    face_off = np.zeros(E + 1, dtype=np.int64)
    np.cumsum(np.maximum(counts - 1, 0), out=face_off[1:])
    # interior faces k = 1 .. counts[e]-1 of every edge at x = k dx[e], the
    # reference's np.arange(1, n) * dx per edge (fvm.py:99-103), all at once
    n_faces = int(face_off[-1])
    face_edge = np.repeat(np.arange(E, dtype=np.int64), np.maximum(counts - 1, 0))
    face_k = (np.arange(n_faces, dtype=np.int64) - face_off[face_edge] + 1).astype(np.float64)
    face_mu = (_drift_pairs(field, face_edge, face_k * dx[face_edge]) if n_faces
               else np.zeros(0, dtype=np.float64))
    sig = np.array([d.at(0.0) for d in field.diffusion], dtype=np.float64)
    D_edge = 0.5 * sig ** 2
    # vertex slots, vectorised over the graph's CSR (slot order = incidence order)
    v_off = np.asarray(graph.v_off, np.int64).copy()
    ve = np.asarray(graph.v_edges, np.int64)
    at_init = np.asarray(graph.v_orient) == AT_INIT
    v_cells = np.where(at_init, offs[ve], offs[ve + 1] - 1).astype(np.int64)
    x_v = np.where(at_init, 0.0, np.asarray(grid.lengths, np.float64)[ve])
    mu_v = _drift_pairs(field, ve, x_v)
    speed = np.where(at_init, -mu_v, mu_v)
    v_speed_in = np.where(speed > 0.0, speed, 0.0)
    v_D = 0.5 * sig[ve] ** 2
    v_b = np.asarray(graph.v_weights, np.float64).copy()
    v_dx = dx[ve]
    deg = np.diff(v_off)
    slot_vertex = np.repeat(np.arange(deg.shape[0], dtype=np.int64), deg)
    multi = deg[slot_vertex] >= 2
    bad = np.unique(slot_vertex[multi & (v_b <= 0.0)])
    if bad.size:
        raise _zero_weight(int(bad[0]))
    n_cells = int(counts.sum())
    owners = np.bincount(v_cells[multi], minlength=n_cells)
    shared = np.zeros(deg.shape[0], dtype=bool)
    shared[np.unique(slot_vertex[multi & (owners[v_cells] >= 2)])] = True
    hub = deg >= 2
    pslot = np.flatnonzero((hub & ~shared)[slot_vertex]).astype(np.int64)
    tstart, rstart, rpos, n_terms = _term_layout(v_off, v_b, v_speed_in, pslot, slot_vertex)
    cell_edge = np.repeat(np.arange(E, dtype=np.int64), counts)
    local = np.arange(n_cells, dtype=np.int64) - offs[cell_edge]
    left = local > 0
    right = local + 1 < counts[cell_edge]
    # face k of edge e (between its cells k and k+1) sits at face_mu[face_off[e] + k]
    fidx = face_off[cell_edge] + local
    cell_mu_l = np.zeros(n_cells)
    cell_mu_r = np.zeros(n_cells)
    cell_mu_l[left] = face_mu[fidx[left] - 1]
    cell_mu_r[right] = face_mu[fidx[right]]
    owned = owners >= 1
    flags = (left.astype(np.uint8) | (right.astype(np.uint8) << 1)
             | (owned.astype(np.uint8) << 2))
    return _Packed(
        offs=offs, dx_edge=dx, D_edge=D_edge, face_mu=face_mu, face_off=face_off, v_off=v_off,
        v_cells=v_cells, v_b=v_b, v_dx=v_dx, v_speed_in=v_speed_in, v_D=v_D,
        cell_edge=cell_edge, owned=owned.astype(np.uint8),
        vpar=np.flatnonzero(hub & ~shared).astype(np.int64),
        vser=np.flatnonzero(hub & shared).astype(np.int64),
        slot_vertex=slot_vertex, pslot=pslot, tstart=tstart, rstart=rstart, rpos=rpos,
        n_terms=n_terms,
        cell_mu_l=cell_mu_l, cell_mu_r=cell_mu_r, cell_D=D_edge[cell_edge].copy(),
        cell_dx=dx[cell_edge].copy(), cell_flags=flags.astype(np.uint8))


def _vertex_template(n: int, active):
    """Term layout of ONE vertex of degree n (the ``active`` drift rows), relative
    to the vertex's first term: (tstart offsets [n], row position lists [n])."""
    tstart = [0] * n
    pos = 0
    where = {}
    for k in range(n):
        tstart[k] = pos
        for i in range(n):
            if active[i]:
                if i == k:
                    for j in range(n):
                        if j != k:
                            where[("o", i, j)] = pos
                            pos += 1
                else:
                    where[("n", i, k)] = pos
                    pos += 1
            if i < k:
                where[("j", i, k)] = pos
                pos += 1
            elif i == k:
                for j in range(k + 1, n):
                    where[("i", k, j)] = pos
                    pos += 1
    rows = []
    for i in range(n):
        r = []
        if active[i]:
            for j in range(n):
                if j != i:
                    r += [where[("n", i, j)], where[("o", i, j)]]
        for j in range(i + 1, n):
            r += [where[("j", i, j)], where[("i", i, j)]]
        rows.append(r)
    return tstart, rows, pos


def _term_layout(v_off, v_b, v_speed_in, pslot, slot_vertex, bitkey=True):
    """Static layout of the two-phase vertex exchange on the GPU.

    Every contribution the reference's exchange loop (``fvm.py:305-328``) adds to
    a vertex-adjacent cell is one signed *term*.  Phase A (one thread per slot
    i = exchange *row*) computes row i's terms -- drift exports i -> j and the
    diffusion pairs (i, j > i) -- and writes each to its position; phase B (one
    thread per slot k) adds the terms of cell k in exactly the order the
    reference applies them:

        for i in 0..n-1:
            drift row i (sp_i > 0 and 1 - b_i > 0):  i == k: -(dt f_ij / dx_i) for j != k
                                                      i != k: +(dt f_ik / dx_k)
            diffusion:  i < k: pair (i, k), k's share;  i == k: pairs (k, j > k), k's share

    so a - b is added as a + (-b), bit-identical.  Returns (tstart, rstart,
    rpos, n_terms): cell k's terms are ``T[tstart[t]:tstart[t+1]]`` (t = its
    index in ``pslot``); row t writes its j-side / i-side pairs to
    ``rpos[rstart[t]:rstart[t+1]]``.  Vertices of equal degree and drift-row
    pattern share one template (``_vertex_template``), placed with numpy."""
    n_p = pslot.shape[0]
    tstart = np.zeros(n_p + 1, dtype=np.int64)
    rstart = np.zeros(n_p + 1, dtype=np.int64)
    if n_p == 0:
        return tstart, rstart, np.zeros(0, dtype=np.int64), 0
    # the vertices in pslot order (each contributes its n consecutive slots)
    first = np.flatnonzero(np.r_[True, slot_vertex[pslot[1:]] != slot_vertex[pslot[:-1]]])
    verts = slot_vertex[pslot[first]]
    lo = np.asarray(v_off, np.int64)[verts]
    deg = np.asarray(v_off, np.int64)[verts + 1] - lo
    act = (np.asarray(v_speed_in) > 0.0) & (1.0 - np.asarray(v_b) > 0.0)
    # per vertex: a key (degree, active-row bits) -> one shared template
    slot_v = np.repeat(np.arange(verts.shape[0], dtype=np.int64), deg)
    local = np.arange(slot_v.shape[0], dtype=np.int64) - np.repeat(base_slot := np.r_[0, np.cumsum(deg)[:-1]], deg)
    gslot = lo[slot_v] + local  # graph slot of every (vertex, local index)
    if bitkey and int(deg.max()) <= 60:
        bits = np.zeros(verts.shape[0], dtype=np.int64)
        np.add.at(bits, slot_v, act[gslot].astype(np.int64) << local)
        code = (bits << 6) | deg
        uniq, kid = np.unique(code, return_inverse=True)
        tmpl = []
        for cval in uniq.tolist():
            n, b = cval & 63, cval >> 6
            tmpl.append(_vertex_template(n, [bool((b >> i) & 1) for i in range(n)]))
    else:  # (hubs wider than the bit key: a key per vertex pattern)
        keys = {}
        kid = np.empty(verts.shape[0], dtype=np.int64)
        for q in range(verts.shape[0]):
            n = int(deg[q])
            a = tuple(bool(x) for x in act[lo[q]:lo[q] + n])
            kid[q] = keys.setdefault((n, a), len(keys))
        tmpl = [None] * len(keys)
        for (n, a), t in keys.items():
            tmpl[t] = _vertex_template(n, list(a))
    kid = np.asarray(kid, dtype=np.int64).reshape(-1)
    keys = range(len(tmpl))
    n_terms_v = np.array([t[2] for t in tmpl], dtype=np.int64)[kid]
    base = np.zeros(verts.shape[0] + 1, dtype=np.int64)
    np.cumsum(n_terms_v, out=base[1:])
    rlen = np.zeros(n_p, dtype=np.int64)
    rpos = [None] * len(keys)
    for t in range(len(keys)):
        sel = np.flatnonzero(kid == t)
        if not sel.size:
            continue
        ts, rows, _ = tmpl[t]
        n = len(ts)
        slots = first[sel][:, None] + np.arange(n)[None, :]  # pslot indices
        tstart[slots] = base[sel][:, None] + np.asarray(ts, np.int64)[None, :]
        rlen[slots] = np.asarray([len(r) for r in rows], np.int64)[None, :]
        rpos[t] = (sel, slots, np.concatenate([np.asarray(r, np.int64) for r in rows])
                   if any(rows) else np.zeros(0, np.int64))
    tstart[n_p] = base[-1]
    np.cumsum(rlen, out=rstart[1:])
    out = np.empty(int(rstart[-1]), dtype=np.int64)
    for t in range(len(keys)):
        if rpos[t] is None:
            continue
        sel, slots, flat = rpos[t]
        if not flat.size:
            continue
        # row positions of slot slots[q, i] start at rstart[slots[q, i]]; one
        # vertex's rows are consecutive, so its flat template lands at rstart[first]
        dst = rstart[slots[:, 0]][:, None] + np.arange(flat.size)[None, :]
        out[dst] = base[sel][:, None] + flat[None, :]
    return tstart, rstart, out, int(base[-1])


def stability_limit(graph: MetricGraph, field: CoefficientField, grid: EdgeGrid) -> float:
    """Largest dt the explicit stepper accepts, CFL = 1 (``fvm.py:209-251``),
    vectorised with the reference's per-element arithmetic and summation order."""
    E = grid.n_edges
    counts = np.asarray(grid.counts, np.int64)
    dx_e = np.asarray(grid.dx, np.float64)
    kind, coef, _, _, _, _ = field.packed()
    kind = np.asarray(kind)
    coef = np.asarray(coef, np.float64)
    # edges: max |mu| over the cell faces x = k dx, k = 0 .. counts (constant:
    # |c|; linear: |c x| grows with x, so the last face; tabulated: scanned)
    x_end = counts.astype(np.float64) * dx_e
    mu_max = np.where(kind == 1, np.abs(coef * x_end), np.abs(coef))
    for e in np.flatnonzero(kind == 2).tolist():
        xs = np.arange(int(counts[e]) + 1) * float(dx_e[e])
        mu_max[e] = float(np.max(np.abs(_drift_at(field, e, xs))))
    sig = np.array([d.at(0.0) for d in field.diffusion], dtype=np.float64)
    D = 0.5 * sig ** 2
    rate_e = mu_max / dx_e + 2.0 * D / (dx_e * dx_e)
    max_rate = max(0.0, float(rate_e.max())) if E else 0.0
    # vertices of degree >= 2: every slot i, the diffusion rates summed over the
    # other slots j in ascending order (the reference's loop order)
    p = _pack(graph, field, grid)
    v_off = np.asarray(p.v_off, np.int64)
    deg = np.diff(v_off)
    hub = np.flatnonzero(deg >= 2)
    if hub.size:
        n_s = deg[hub]
        lo_s = np.repeat(v_off[hub], n_s)
        n_i = np.repeat(n_s, n_s)
        i = lo_s + (np.arange(lo_s.shape[0]) - np.repeat(np.r_[0, np.cumsum(n_s)[:-1]], n_s))
        b, dxs, D_v = p.v_b, p.v_dx, p.v_D
        diff_rate = np.zeros(i.shape[0])
        for jj in range(int(n_s.max())):
            j = lo_s + jj
            m = (jj < n_i) & (j != i)
            if not m.any():
                continue
            im, jm = i[m], j[m]
            dxh = 2.0 * dxs[im] * dxs[jm] / (dxs[im] + dxs[jm])
            diff_rate[m] = diff_rate[m] + D_v[im] * b[jm] / (b[im] * dxh)
        eid = np.asarray(graph.v_edges, np.int64)[i]
        x_v = np.where(np.asarray(graph.v_orient)[i] == AT_INIT, 0.0,
                       np.asarray(grid.lengths, np.float64)[eid])
        mu_abs = np.abs(_drift_pairs(field, eid, x_v))
        dx = dxs[i]
        rate = (p.v_speed_in[i] / dx + diff_rate / dx + mu_abs / dx + 2.0 * D_v[i] / (dx * dx))
        max_rate = max(max_rate, float(rate.max()))
    if max_rate == 0.0:
        return math.inf
    return 1.0 / max_rate


_DESC_ARRAYS = ("cell_mu_l", "cell_mu_r", "cell_D", "cell_dx", "cell_flags", "v_off", "v_cells",
                "v_b", "v_dx", "v_speed_in", "v_D", "slot_vertex", "pslot", "vser", "tstart",
                "rstart", "rpos")


class _Desc(C.Structure):
    """``gsde_fvm_desc`` (include/gsde.h)."""

    _fields_ = [(n, C.c_int64) for n in ("n_edges", "n_cells", "n_vertices", "n_pslot", "n_vser",
                                         "n_terms")] + [
        (n, C.c_void_p) for n in _DESC_ARRAYS + ("terms",)]


def _device_pack(p: _Packed, n_vertices: int, device: int):
    torch, dev = _native.torch_cuda(device)
    kw = dict(device=f"cuda:{dev}")
    keep = {}
    d = _Desc()
    d.n_edges, d.n_cells = p.dx_edge.shape[0], p.cell_edge.shape[0]
    d.n_vertices, d.n_pslot, d.n_vser = n_vertices, p.pslot.shape[0], p.vser.shape[0]
    d.n_terms = p.n_terms
    for name in _DESC_ARRAYS:
        a = getattr(p, name)
        t = torch.from_numpy(np.ascontiguousarray(a) if a.size else np.zeros(1, a.dtype)).to(**kw)
        keep[name] = t
        setattr(d, name, t.data_ptr())
    keep["terms"] = torch.empty(max(1, p.n_terms), dtype=torch.float64, **kw)  # workspace
    d.terms = keep["terms"].data_ptr()
    return d, keep, torch, dev


def fvm_run(graph: MetricGraph, field: CoefficientField, grid: EdgeGrid, dt: float,
            n_steps: int, initial: FvmState, force: bool = False) -> FvmResult:
    """Advance the density ``n_steps`` explicit Euler steps of size ``dt`` (``fvm.py:385-422``).

    Raises :class:`UnstableTimestep` when the predicted CFL number exceeds 1
    unless ``force``; a developing negative density raises
    :class:`NegativeDensity`.  The steps run on the GPU (bit-identical to the
    reference stepper)."""
    if not dt > 0.0:
        raise ValueError(f"dt must be positive, got {dt!r}")
    if not initial.grid.same_geometry(grid):
        raise ValueError("initial state lives on a different grid")
    limit = stability_limit(graph, field, grid)
    max_cfl = dt / limit if math.isfinite(limit) else 0.0
    if max_cfl > 1.0 and not force:
        raise UnstableTimestep(
            f"dt={dt:g} exceeds the stability limit {limit:g} (CFL={max_cfl:.3g}); "
            "pass force=True to run anyway")
    state = initial.copy()
    rho, neg = fvm_steps_device(graph, field, grid, state.rho, int(n_steps), float(dt))
    state.rho = rho
    if neg:
        state.t += neg * dt
        raise NegativeDensity(
            f"density went negative at t={state.t:g} (step {neg}); the timestep is unstable")
    state.t += n_steps * dt
    return FvmResult(state=state, max_cfl=max_cfl, n_steps=int(n_steps))


class FvmDevice:
    """A (graph, field, grid) packed and resident on one GPU; ``run`` steps a
    device density in place (the whole run is one kernel launch)."""

    def __init__(self, graph, field, grid, device=None):
        self.packed = _pack(graph, field, grid)
        self.desc, self._keep, self.torch, self.device = _device_pack(
            self.packed, graph.n_vertices, device)
        self.n_cells = self.packed.cell_edge.shape[0]
        t = self.torch
        self._scratch = t.empty(self.n_cells, dtype=t.float64, device=f"cuda:{self.device}")
        self._red = t.zeros(8, dtype=t.int64, device=f"cuda:{self.device}")

    def run(self, rho, n_steps: int, dt: float, stream=None):
        """Advance the device tensor ``rho`` in place; returns a device int64[1]
        holding the 1-based negative-density step (0 = none)."""
        t = self.torch
        if rho.dtype != t.float64 or rho.numel() != self.n_cells or not rho.is_contiguous():
            raise ValueError("rho must be a contiguous float64 tensor with one value per cell")
        neg = t.zeros(1, dtype=t.int64, device=rho.device)
        s = stream if stream is not None else _native.cur_stream(self.device)
        _native.check(_native.lib().gsde_fvm_run(
            C.byref(self.desc), rho.data_ptr(), self._scratch.data_ptr(), int(n_steps), float(dt),
            -_NEGATIVE_TOL, neg.data_ptr(), self._red.data_ptr(), s))
        return neg


def fvm_steps_device(graph, field, grid, rho, n_steps, dt, device=None, stream=None):
    """The stepper alone (no CFL check): returns (rho after the run, 1-based
    negative step or 0).  ``rho`` may be a numpy array (copied to and from the
    device) or a CUDA float64 tensor (updated in place)."""
    fd = FvmDevice(graph, field, grid, device)
    torch = fd.torch
    host = not (hasattr(rho, "is_cuda") and rho.is_cuda)
    r = (torch.from_numpy(np.array(rho, dtype=np.float64, copy=True)).to(f"cuda:{fd.device}")
         if host else rho)
    n = int(fd.run(r, n_steps, dt, stream).item())
    return (r.cpu().numpy() if host else r), n
