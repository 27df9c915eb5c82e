"""Host-side checks of the C-ABI library (no GPU needed): it loads, exports every symbol
include/dock.h declares, validates its inputs, and its D1 preprocessing (host C++)
matches the oracle bit-exactly."""
import ctypes as C
import os
import re

import numpy as np
import pytest

import oracle
from gen import CONFIGS, TYPE_TABLE, config_inputs, hts_ligands, make_ligand
from gen.synth import TYPE_NAMES

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def dock():
    from paper_2203_02096_b200._build import build
    build()
    import paper_2203_02096_b200 as d
    return d


def test_exports_every_declared_symbol(dock):
    hdr = open(os.path.join(ROOT, "include", "dock.h")).read()
    declared = set(re.findall(r"^\s*(?:int|void|int64_t|const char \*)\s*\*?(dock_\w+)\s*\(", hdr, re.M))
    assert len(declared) >= 20
    lib = C.CDLL(dock.LIB_PATH)
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert declared == set(dock.EXPORTED)


def test_introspection_null_context(dock):
    # engine / launch queries on a NULL context: -1, never a crash (include/dock.h)
    assert dock.lib.dock_last_engine(None) == -1
    assert dock.lib.dock_tile_schedule(None) == -1
    assert dock.lib.dock_run_branches(None) == -1
    assert dock.lib.dock_launch_count(None) == -1


def test_params_default(dock):
    p = dock.params_default()
    assert (p.p_tour, p.p_cross, p.p_mut) == (np.float32(0.6), np.float32(0.8), np.float32(0.02))
    assert p.ls_max_iters == 300 and p.max_generations == 27000 and p.gens_per_graph == 16
    assert abs(p.ad_rho - 0.8) < 1e-7 and abs(p.ad_eps - 1e-2) < 1e-9
    # NEXT-2: D5 by default, AD4.1 coefficients filled in for DOCK_SF_AD4
    assert p.scoring == dock.SF_D5
    assert (p.w_vdw, p.w_hb, p.w_el, p.w_ds, p.w_tors, p.qasp) == tuple(
        np.float32(v) for v in (0.1662, 0.1209, 0.1406, 0.1322, 0.2983, 0.01097))


@pytest.mark.parametrize("bad", [dict(scoring=2), dict(scoring=1, w_el=-1.0), dict(scoring=1, qasp=float("nan"))])
def test_scoring_params_validated_before_device(dock, bad):
    from gen import config_inputs
    cfg, lig, grid = config_inputs("tiny")
    with pytest.raises(dock.DockError) as e:
        dock.Docker.from_inputs(grid, lig, **bad)
    assert e.value.code == dock.DOCK_E_INPUT


def test_builtin_table_matches_input_table(dock):
    for name in TYPE_NAMES:
        t = dock.builtin_type_param(name)
        R, eps, S, V, role = TYPE_TABLE[name]
        assert (t.R, t.eps, t.S, t.V, t.role) == (np.float32(R), np.float32(eps), np.float32(S), np.float32(V), role)
    with pytest.raises(dock.DockError):
        dock.builtin_type_param("Xx")


def _topo_dock(dock, lig, grid_types):
    tp = np.array([TYPE_TABLE[t][:4] for t in grid_types], np.float32)
    roles = np.array([TYPE_TABLE[t][4] for t in grid_types], np.int32)
    return dock.topology(lig.types, lig.charges, lig.xyz, lig.bonds, lig.rotatable, tp, roles)


@pytest.mark.parametrize("name", ["tiny", "1stp", "3ce3", "7cpa"])
def test_topology_bit_exact_vs_oracle(dock, name):
    cfg = CONFIGS[name]
    lig = make_ligand(cfg.n_atoms, cfg.n_tors, cfg.lig_seed, type_names=TYPE_NAMES)
    axis, moved, pairs = _topo_dock(dock, lig, TYPE_NAMES)
    ref = oracle.topology(lig.n_atoms, lig.bonds, lig.rotatable)
    assert np.array_equal(pairs, ref["pairs"])
    assert np.array_equal(axis[:, 0], ref["tor_a"]) and np.array_equal(axis[:, 1], ref["tor_b"])
    assert np.array_equal(moved, ref["moved"])


def test_topology_bit_exact_hts_sample(dock):
    for lig in hts_ligands(60, seed=5):
        axis, moved, pairs = _topo_dock(dock, lig, TYPE_NAMES)
        ref = oracle.topology(lig.n_atoms, lig.bonds, lig.rotatable)
        assert np.array_equal(pairs, ref["pairs"])
        assert np.array_equal(axis, np.stack([ref["tor_a"], ref["tor_b"]], 1).reshape(-1, 2))
        assert np.array_equal(moved, ref["moved"])


def test_topology_with_rings_vs_oracle(dock):
    # benzene-like ring with two substituent chains; rotatable bonds are bridges only
    bonds = [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 0), (0, 6), (6, 7), (7, 8), (3, 9), (9, 10), (10, 11)]
    rot = [0, 0, 0, 0, 0, 0, 1, 1, 0, 1, 0, 1]
    n = 12

    class L:
        pass
    lig = L()
    lig.types = np.zeros(n, np.int32); lig.charges = np.zeros(n, np.float32)
    ang = np.arange(n) * 0.7
    lig.xyz = np.stack([np.cos(ang) * 3 + np.arange(n) * 0.1, np.sin(ang) * 3, np.arange(n) * 0.3], 1).astype(np.float32)
    lig.bonds = np.array(bonds, np.int32); lig.rotatable = np.array(rot, np.uint8)
    axis, moved, pairs = _topo_dock(dock, lig, ["C"])
    ref = oracle.topology(n, lig.bonds, lig.rotatable)
    assert np.array_equal(pairs, ref["pairs"]) and np.array_equal(moved, ref["moved"])
    assert np.array_equal(axis[:, 0], ref["tor_a"]) and np.array_equal(axis[:, 1], ref["tor_b"])
    lig.rotatable = np.array([1] + rot[1:], np.uint8)          # a ring bond: rejected
    with pytest.raises(dock.DockError, match="ring"):
        _topo_dock(dock, lig, ["C"])


def test_init_validation_errors(dock):
    cfg, lig, grid = config_inputs("tiny")
    bad = lig.types.copy(); bad[3] = 99
    with pytest.raises(dock.DockError) as e:
        tp, roles = grid.type_params()
        dock.Docker(grid.maps, grid.n, grid.spacing, grid.origin, tp, roles, bad, lig.charges, lig.xyz,
                    lig.bonds, lig.rotatable)
    assert e.value.code == dock.DOCK_E_INPUT and "type[3]" in str(e.value)
    with pytest.raises(dock.DockError) as e:
        dock.Docker(grid.maps, grid.n, -1.0, grid.origin, tp, roles, lig.types, lig.charges, lig.xyz,
                    lig.bonds, lig.rotatable)
    assert e.value.code == dock.DOCK_E_INPUT and "spacing" in str(e.value)
    maps = grid.maps.copy(); maps[0, 1, 2, 3] = np.nan
    with pytest.raises(dock.DockError, match="non-finite"):
        dock.Docker(maps, grid.n, grid.spacing, grid.origin, tp, roles, lig.types, lig.charges, lig.xyz,
                    lig.bonds, lig.rotatable)
    with pytest.raises(dock.DockError, match="probabilities"):
        dock.Docker.from_inputs(grid, lig, p_mut=1.5)


def test_no_cpu_fallback_without_gpu(dock):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    cfg, lig, grid = config_inputs("tiny")
    with pytest.raises(dock.DockError) as e:
        dock.Docker.from_inputs(grid, lig)
    assert e.value.code == dock.DOCK_E_INTERNAL


def test_builtin_types_need_names_and_known_names(dock):
    """dock_init with NULL type_params: the built-in table by grids.type_names;
    missing / unknown / duplicate names are input errors, raised before any device use."""
    from gen import config_inputs
    cfg, lig, grid = config_inputs("tiny")
    with pytest.raises(dock.DockError):
        dock.Docker(grid.maps, grid.n, grid.spacing, grid.origin, None, None, lig.types, lig.charges, lig.xyz,
                    lig.bonds, lig.rotatable)
    bad = list(grid.type_names)
    bad[0] = "Zz"
    with pytest.raises(dock.DockError) as e:
        dock.Docker(grid.maps, grid.n, grid.spacing, grid.origin, None, None, lig.types, lig.charges, lig.xyz,
                    lig.bonds, lig.rotatable, type_names=bad)
    assert e.value.code == dock.DOCK_E_INPUT
    dup = list(grid.type_names)
    dup[1] = dup[0]
    tp, roles = grid.type_params()
    with pytest.raises(dock.DockError):
        dock.Docker(grid.maps, grid.n, grid.spacing, grid.origin, tp, roles, lig.types, lig.charges, lig.xyz,
                    lig.bonds, lig.rotatable, type_names=dup)
