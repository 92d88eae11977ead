"""The C-ABI library loads and exports exactly what include/gsde.h declares
(CPU; no compute calls need a GPU)."""

import ctypes as C
import os
import re

import numpy as np
import pytest

import golden_io
from paper_2512_02175_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "gsde.h")).read()
    return sorted(set(re.findall(r"\b(gsde_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert sorted(_native.EXPORTS) == declared_symbols()


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_native.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.gsde_abi_version() == 3


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_native.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out, out


def test_host_helpers_match_reference_vectors():
    L = _native.lib()
    for row in golden_io.load_json("rng.json")["raw64_grid"]:
        s, st, k = int(row["seed"]), int(row["stream"]), int(row["index"])
        assert L.gsde_raw64(s, st, k) == int(row["raw"])
        assert L.gsde_uniform01(s, st, k) == row["uniform"]
    for row in golden_io.load_json("solvers.json")["first_passage"]:
        s = L.gsde_solve_first_passage_s(row["a"], row["b"], row["c"])
        assert s == row["s"] or abs(s - row["s"]) <= 1e-13 * max(abs(s), abs(row["s"]))


def test_error_paths_without_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("checks the no-device error path")
    L = _native.lib()
    d = _native.GraphDesc()
    h = C.c_void_p()
    assert L.gsde_graph_create(None, 0, C.byref(h)) == -1
    rc = L.gsde_graph_create(C.byref(d), 0, C.byref(h))
    assert rc in (-1, -4)
    assert L.gsde_ensemble(None, None, None, None) == -1
    assert b"null" in L.gsde_last_error()
    with pytest.raises(_native.NativeUnavailable):
        _native.torch_cuda()


def test_product_path_fails_loudly_without_gpu():
    import torch

    import cases
    import paper_2512_02175_b200 as gs

    if torch.cuda.is_available():
        pytest.skip("no-GPU behaviour")
    g, f = cases.build("star3_bm", gs)
    with pytest.raises(_native.NativeUnavailable):
        gs.run_ensemble(g, f, gs.SimulationConfig(dt=1e-3, n_steps=1, n_particles=4, seed=1))
    with pytest.raises(_native.NativeUnavailable):
        gs.analysis.histogram_accumulate(np.zeros(2, np.int64), np.zeros(2),
                                         gs.EdgeGrid.uniform(g, 2, lengths=[1.0] * 3))


def test_integration_stub_structs_match_the_abi():
    """The ctypes stub in INTEGRATION.md (what a reference maintainer would paste)
    declares every field of gsde_graph_desc / gsde_run / gsde_out, in order."""
    import ast
    import os
    import re

    from paper_2512_02175_b200 import _native

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    text = open(os.path.join(root, "INTEGRATION.md")).read()
    for stub, ours in (("GraphDesc", _native.GraphDesc), ("Run", _native.Run),
                       ("Out", _native.Out)):
        m = re.search(r"class %s\(C\.Structure\):\s*_fields_ = (\[.*?\])[ \t]*(?:#[^\n]*)?\n"
                      % stub, text, re.S)
        assert m, stub
        src = re.sub(r"#[^\n]*", "", m.group(1))
        names = [n for n, _ in ast.literal_eval(re.sub(r"\b(P|i64|u64|f64|i32)\b", "0", src))]
        assert names == [f[0] for f in ours._fields_], stub
