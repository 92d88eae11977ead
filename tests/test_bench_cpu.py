"""bench.py contract on the CPU: the reference arm (the reference's own numba
path from baseline/_ref, or the oracle port when that is not installed; no
GPU) prints one JSON line with the keys the driver reads."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["cores"] >= 1
    if os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "graphsde")):
        assert d["cpu_baseline"]["kind"] == "reference", d
        assert "graphsde.run_ensemble" in d["config"]["sample"]
    else:
        assert d["cpu_baseline"]["kind"] == "port" and "reference_unavailable" in d
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert "workload" in d["config"]


def _ref_or_skip():
    import pytest

    sys.path.insert(0, ROOT)
    import bench

    R, why = bench.reference_package()
    if R is None:
        pytest.skip(why)
    return R


def test_reference_arm_builds_identical_graphs():
    """The reference arm times the reference on the same graphs: built through
    the reference's own constructors / graph-file parser, their packed arrays
    equal this package's."""
    import numpy as np

    import paper_2512_02175_b200 as gs
    from paper_2512_02175_b200 import workloads

    R = _ref_or_skip()
    for make in (workloads.star3, workloads.hub64, workloads.star5,
                 lambda api=None: workloads.vascular(3000, api=api)):
        g1, f1 = make()
        g2, f2 = make(api=R)
        for k in ("edge_length", "edge_init", "edge_term", "v_off", "v_edges", "v_orient",
                  "v_cumw"):
            np.testing.assert_array_equal(getattr(g1, k), getattr(g2, k), err_msg=k)
        for a, b in zip(f1.packed(), f2.packed()):
            np.testing.assert_array_equal(a, b)
        assert g1.is_star == g2.is_star
    assert isinstance(gs.workloads.star3()[0], gs.MetricGraph)
