"""Streamed results (gsde_out.progress + gsde_stream_wait_geq32): run_ensemble's
host arrays from ONE launch whose per-particle outputs are copied range by
range while it runs must equal the device arrays of a plain launch and the
chunked-launch pipeline, bit for bit."""
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import _native, engine, workloads

pytestmark = pytest.mark.gpu

NAMES = ("edge", "x", "crossings", "events")


def _graphs():
    g, f = workloads.star3()
    yield "star3", g, f, gs.AtVertex(0)
    g, f = workloads.hub64()
    yield "hub64", g, f, gs.PerEdgeUniform(2.0)
    g, f = workloads.vascular(20_000, seed=5)
    yield "vasc", g, f, gs.PerEdgeUniform(float(g.edge_length.max()))


@pytest.mark.parametrize("n, n_steps", [(300_001, 40), (70_000, 200)])
def test_streamed_pipeline_equals_plain_launch(monkeypatch, n, n_steps):
    import torch

    monkeypatch.setattr(engine, "_PIPELINE_MIN", 1)
    calls = []
    real = engine._streamed_to_host
    monkeypatch.setattr(engine, "_streamed_to_host", lambda *a, **k: calls.append(1) or real(*a, **k))
    for name, g, f, init in _graphs():
        cfg = gs.SimulationConfig(dt=1e-3, n_steps=n_steps, n_particles=n, seed=11,
                                  initial=init)
        plain = engine.ensemble_device(g, f, cfg, outputs=NAMES)
        torch.cuda.synchronize()
        want = [plain[k].cpu().numpy() for k in NAMES]
        want_m = plain["m_hist"].cpu().numpy()
        want_t = plain["totals"].cpu().numpy()
        before = len(calls)
        got = engine._ensemble_to_host(g, f, cfg)
        assert len(calls) == before + 1, "the streamed path did not run"
        for k, a, b in zip(NAMES, want, got[:4]):
            np.testing.assert_array_equal(a, b, err_msg=f"{name} {k}")
        np.testing.assert_array_equal(want_m, got[4])
        np.testing.assert_array_equal(want_t, got[5])
        monkeypatch.setenv("GSDE_NO_STREAMING", "1")  # the chunked pipeline agrees too
        chunked = engine._ensemble_to_host(g, f, cfg)
        monkeypatch.delenv("GSDE_NO_STREAMING")
        assert len(calls) == before + 1
        for k, a, b in zip(NAMES + ("m_hist", "totals"), got, chunked):
            np.testing.assert_array_equal(a, b, err_msg=f"{name} chunked {k}")


@pytest.mark.parametrize("shift", [0, 5, 12])
def test_progress_counts_every_particle_once(shift):
    import torch

    g, f = workloads.hub64()
    n = 100_003
    cfg = gs.SimulationConfig(dt=1e-3, n_steps=30, n_particles=n, seed=2,
                              initial=gs.PerEdgeUniform(2.0))
    n_ranges = ((n - 1) >> shift) + 1
    prog = torch.zeros(n_ranges, dtype=torch.int32, device="cuda")
    engine.ensemble_device(g, f, cfg, outputs=("edge",), progress=(prog, shift))
    want = np.full(n_ranges, 1 << shift)
    want[-1] = n - ((n_ranges - 1) << shift)
    np.testing.assert_array_equal(prog.cpu().numpy(), want)
    # placement only (n_steps = 0) publishes too
    prog.zero_()
    cfg0 = gs.SimulationConfig(dt=1e-3, n_steps=0, n_particles=n, seed=2,
                               initial=gs.PerEdgeUniform(2.0))
    engine.ensemble_device(g, f, cfg0, outputs=("x",), progress=(prog, shift))
    np.testing.assert_array_equal(prog.cpu().numpy(), want)


def test_progress_rejected_where_it_does_not_apply():
    import torch

    g, f = workloads.hub64()
    prog = torch.zeros(4, dtype=torch.int32, device="cuda")
    ref = gs.SimulationConfig(dt=1e-3, n_steps=5, n_particles=1000, seed=2, rng="reference",
                              initial=gs.PerEdgeUniform(2.0))
    with pytest.raises(_native.GsdeError):
        engine.ensemble_device(g, f, ref, outputs=("edge",), progress=(prog, 8))
    nat = gs.SimulationConfig(dt=1e-3, n_steps=5, n_particles=1000, seed=2,
                              initial=gs.PerEdgeUniform(2.0))
    with pytest.raises(_native.GsdeError):  # no per-particle output to count
        engine.ensemble_device(g, f, nat, outputs=("edge_counts",), progress=(prog, 8))
    with pytest.raises(_native.GsdeError):
        engine.ensemble_device(g, f, nat, outputs=("edge",), progress=(prog, 63))


_CHUNKED_PROGRESS = r"""
import sys
sys.path.insert(0, {root!r})
import numpy as np, torch
import paper_2512_02175_b200 as gs
from paper_2512_02175_b200 import engine, workloads
g, f = workloads.hub64()
n, shift = 100_003, 10
cfg = gs.SimulationConfig(dt=1e-3, n_steps=30, n_particles=n, seed=2,
                          initial=gs.PerEdgeUniform(2.0))
prog = torch.zeros(((n - 1) >> shift) + 1, dtype=torch.int32, device="cuda")
r = engine.ensemble_device(g, f, cfg, outputs=("edge", "x"), progress=(prog, shift))
np.savez({path!r}, prog=prog.cpu().numpy(), edge=r["edge"].cpu().numpy(), x=r["x"].cpu().numpy())
"""


def test_progress_base_across_internal_chunks(tmp_path):
    """gsde_ensemble's internal particle-id chunks (GSDE_CHUNK_PARTICLES forces
    7777-particle launches) offset each launch's counters by its first id."""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = {}
    for chunk in (None, "7777"):
        path = str(tmp_path / f"p_{chunk}.npz")
        env = dict(os.environ)
        env.pop("GSDE_CHUNK_PARTICLES", None)
        if chunk:
            env["GSDE_CHUNK_PARTICLES"] = chunk
        subprocess.run([sys.executable, "-c", _CHUNKED_PROGRESS.format(root=root, path=path)],
                       check=True, env=env, timeout=600)
        out[chunk] = np.load(path)
    a, b = out[None], out["7777"]
    n, shift = 100_003, 10
    want = np.full(len(a["prog"]), 1 << shift)
    want[-1] = n - ((len(want) - 1) << shift)
    np.testing.assert_array_equal(a["prog"], want)
    np.testing.assert_array_equal(b["prog"], want)
    np.testing.assert_array_equal(a["edge"], b["edge"])
    np.testing.assert_array_equal(a["x"], b["x"])


def test_kernel_bound_runs_keep_chunked_launches(monkeypatch):
    """n_steps >= 256: the chunked pipeline (measured faster there)."""
    monkeypatch.setattr(engine, "_PIPELINE_MIN", 1)
    monkeypatch.setattr(engine, "_streamed_to_host",
                        lambda *a, **k: pytest.fail("streamed path on a kernel-bound run"))
    g, f = workloads.star3()
    cfg = gs.SimulationConfig(dt=1e-3, n_steps=300, n_particles=50_000, seed=1,
                              initial=gs.AtVertex(0))
    engine._ensemble_to_host(g, f, cfg)


def test_streamed_shard_equals_plain_shard(monkeypatch):
    """A rank's shard (global-id offset, as parallel.run_ensemble_distributed
    asks for it) streams like the whole run: progress ranges are launch-relative."""
    import torch

    monkeypatch.setattr(engine, "_PIPELINE_MIN", 1)
    g, f = workloads.vascular(20_000, seed=5)
    cfg = gs.SimulationConfig(dt=1e-3, n_steps=60, n_particles=1_000_000, seed=8,
                              initial=gs.PerEdgeUniform(float(g.edge_length.max())))
    off, n = 123_457, 300_001
    plain = engine.ensemble_device(g, f, cfg, pid_offset=off, n_particles=n, outputs=NAMES)
    torch.cuda.synchronize()
    got, est = engine._ensemble_to_host(g, f, cfg, pid_offset=off, n_particles=n,
                                        estimators=True)
    for k, b in zip(NAMES, got):
        np.testing.assert_array_equal(plain[k].cpu().numpy(), b, err_msg=k)
    np.testing.assert_array_equal(plain["m_hist"].cpu().numpy(), est["m_hist"].cpu().numpy())
