"""NEXT-3 result serialisation (dock_write_result, host-only C++): JSON and
CSV round trips, the overall-best rule (minimum over runs, NaN as +inf, lowest run on
ties), optional columns, empty timing table."""
import csv
import io
import json
import math

import numpy as np
import pytest


@pytest.fixture(scope="module")
def dock():
    from paper_2203_02096_b200._build import build
    build()
    import paper_2203_02096_b200 as d
    return d


def result(R=10, N=5, G=9, seed=0):
    rng = np.random.default_rng(seed)
    return dict(best_E=rng.normal(-5, 2, R).astype(np.float32), best_genes=rng.normal(0, 1, (R, G)).astype(np.float32),
                best_xyz=rng.normal(0, 3, (R, N, 3)).astype(np.float32), evals=rng.integers(1000, 9000, R),
                generations=rng.integers(1, 50, R).astype(np.int32), cluster=rng.integers(0, 3, R).astype(np.int32),
                rmsd_to_seed=rng.uniform(0, 2, R).astype(np.float32), dG=rng.normal(-3, 1, R).astype(np.float32))


def test_json_round_trip_exact(dock):
    r = result()
    t = dock.write_result(r, "json", timings={"k_ls_adadelta": 12.5, "k_ga": 0.25})
    j = json.loads(t)
    b = int(np.argmin(r["best_E"]))
    assert j["best_run"] == b and np.float32(j["best_energy"]) == r["best_E"][b]
    assert np.array_equal(np.array(j["best_genotype"], np.float32), r["best_genes"][b])
    assert np.array_equal(np.array(j["best_coordinates"], np.float32), r["best_xyz"][b])
    assert len(j["per_run"]) == 10
    for i, row in enumerate(j["per_run"]):
        assert row["run"] == i and np.float32(row["best_energy"]) == r["best_E"][i]
        assert row["evals"] == r["evals"][i] and row["generations"] == r["generations"][i]
        assert row["cluster"] == r["cluster"][i] and np.float32(row["dG"]) == r["dG"][i]
    sizes = {c["id"]: c["size"] for c in j["clusters"]}
    for c, n in sizes.items():
        assert n == int((r["cluster"] == c).sum())
    for c in j["clusters"]:
        members = np.flatnonzero(r["cluster"] == c["id"])
        assert c["best_run"] == members[np.argmin(r["best_E"][members])]
    assert j["timings"] == {"k_ls_adadelta": 12.5, "k_ga": 0.25}


def test_csv_rows_and_json_csv_agree(dock):
    r = result(R=10)
    rows = list(csv.DictReader(io.StringIO(dock.write_result(r, "csv"))))
    assert len(rows) == 10
    j = json.loads(dock.write_result(r, "json"))
    for row, jr in zip(rows, j["per_run"]):
        assert np.float32(float(row["best_energy"])) == np.float32(jr["best_energy"])
        assert int(row["evals"]) == jr["evals"] and int(row["cluster"]) == jr["cluster"]


def test_optional_columns_nan_ties_and_empty_timings(dock):
    E = np.array([np.nan, -2.0, -2.0, 1.0], np.float32)
    r = dict(best_E=E, best_genes=np.zeros((4, 7), np.float32))
    j = json.loads(dock.write_result(r, "json"))
    assert j["best_run"] == 1 and j["best_energy"] == -2.0          # NaN as +inf, lowest run on ties
    assert j["per_run"][0]["best_energy"] is None and j["timings"] == {} and j["clusters"] == []
    assert j["best_coordinates"] == [] and "evals" not in j["per_run"][0]
    rows = list(csv.DictReader(io.StringIO(dock.write_result(r, "csv"))))
    assert rows[0]["best_energy"] == "" and rows[1]["evals"] == "" and len(rows) == 4
    all_nan = dict(best_E=np.full(2, np.nan, np.float32), best_genes=np.zeros((2, 6), np.float32))
    assert json.loads(dock.write_result(all_nan, "json"))["best_run"] == 0
    empty = dict(best_E=np.zeros(0, np.float32), best_genes=np.zeros((0, 6), np.float32))
    je = json.loads(dock.write_result(empty, "json"))
    assert je["best_run"] == -1 and je["best_energy"] is None and je["per_run"] == []


def test_float32_values_round_trip_through_text(dock):
    vals = np.array([1e-38, -3.4028235e38, 0.1, -123.456789, 7.0, -0.0], np.float32)
    r = dict(best_E=vals, best_genes=np.zeros((6, 6), np.float32))
    j = json.loads(dock.write_result(r, "json"))
    got = np.array([p["best_energy"] for p in j["per_run"]], np.float32)
    assert np.array_equal(got.view(np.uint32)[:5], vals.view(np.uint32)[:5]) and got[5] == 0.0


def test_screen_table_json_csv(dock):
    rng = np.random.default_rng(2)
    n = 7
    out = dict(best_E=rng.normal(-5, 2, n).astype(np.float32), best_run=rng.integers(0, 10, n).astype(np.int32),
               best_genes=rng.normal(0, 1, (n, 38)).astype(np.float32), evals=rng.integers(1000, 9000, n),
               status=np.array([0, 0, 1, 0, 0, 0, 0], np.int32), device=np.zeros(n, np.int32))
    out["best_E"][2] = np.nan
    out["best_E"][5] = -20.0
    out["status"][5] = 1                                   # rejected ligand: never the best
    ng = np.full(n, 11, np.int32)
    j = json.loads(dock.write_screen(out, "json", ids=np.arange(100, 107), n_genes=ng))
    ok = [i for i in range(n) if out["status"][i] == 0]
    b = ok[int(np.argmin(out["best_E"][ok]))]
    assert j["best"]["ligand"] == b and np.float32(j["best"]["best_energy"]) == out["best_E"][b]
    assert [r["id"] for r in j["ligands"]] == list(range(100, 107))
    assert j["ligands"][2]["best_energy"] is None and "best_genotype" not in j["ligands"][2]
    assert np.array_equal(np.array(j["ligands"][0]["best_genotype"], np.float32), out["best_genes"][0, :11])
    rows = list(csv.DictReader(io.StringIO(dock.write_screen(out, "csv"))))
    assert len(rows) == n and rows[2]["best_energy"] == "" and int(rows[3]["evals"]) == out["evals"][3]
