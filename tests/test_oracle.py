"""Pin the CPU oracle (oracle/) against the reference's own outputs.

Golden vectors were produced by importing the reference package (see
tests/golden/make_golden.py); these tests run without the reference and
without a GPU.
"""
import gzip
import json
from pathlib import Path

import numpy as np
import pytest

import fuzzgen
import recipes
from oracle import oracle as O

GOLD = Path(__file__).resolve().parent / "golden"


def _run(op, x, y, n_out, r_ps):
    try:
        if op == "minmaxlttb":
            return {"out": O.minmaxlttb(x, y, n_out, r_ps).tolist()}
        if op == "lttb":
            return {"out": O.lttb(x, y, n_out).tolist()}
        if op == "minmax":
            return {"out": O.minmax(y, n_out).tolist()}
        if op == "minmax_preselect":
            return {"out": O.minmax_preselect(y, n_out, r_ps).tolist()}
        if op == "m4":
            return {"out": O.m4(y, n_out).tolist()}
    except O.OracleError as e:
        return {"error": e.name}
    raise ValueError(op)


def test_kats():
    k = json.loads((GOLD / "kats.json").read_text())
    for key, b in k["partition"].items():
        s, e, n = map(int, key.split(","))
        assert O.partition(s, e, n).tolist() == b
    a = [1, 3, 2, 0, 5, 4, 9, 8]
    xa = list(range(8))
    assert O.minmax(a, 4).tolist() == k["minmax"] == k["spec_literal"]["minmax"]
    assert O.m4(a, 8).tolist() == k["m4"] == k["spec_literal"]["m4"]
    assert O.lttb(range(6), [0, 0, 10, 0, 0, 0], 3).tolist() == k["lttb_spike"]
    assert O.minmax([3.0] * 10, 4).tolist() == k["minmax_constant_n10"]
    assert O.lttb(range(20), range(20), 6).tolist() == k["lttb_collinear_n20"]
    assert O.minmax_preselect(np.sin(np.arange(10.0)), 4, 2).tolist() == k["preselect_sin10"]
    assert O.minmaxlttb(xa, a, 4, 1).tolist() == k["minmaxlttb_r1"]
    assert O.minmax([0.0, -0.0, 0.0, -0.0], 4).tolist() == k["signed_zero_minmax"]


def _fuzz():
    with gzip.open(GOLD / "fuzz.json.gz", "rt") as f:
        return json.load(f)


def test_fuzz_cases_regenerate_identically():
    for rec in _fuzz()[::7]:
        c = fuzzgen.make_case(rec["i"])
        assert fuzzgen.digest(c["x"], c["y"]) == rec["digest"]


def test_oracle_matches_reference_on_fuzz():
    bad = []
    for rec in _fuzz():
        c = fuzzgen.make_case(rec["i"])
        got = _run(rec["op"], c["x"], c["y"], rec["n_out"], rec["r_ps"])
        want = {k: rec[k] for k in ("out", "error") if k in rec}
        if got != want:
            bad.append((rec["i"], rec["op"], rec["kind"]))
    assert not bad, bad[:10]


def test_parallel_threads_identical():
    x, y = recipes.c1(200_000)
    ref = O.minmaxlttb(x, y, 1000, 4, threads=1)
    for t in (2, 4, 8):
        assert np.array_equal(O.minmaxlttb(x, y, 1000, 4, threads=t), ref)


def test_typed_chunked_matches_f64():
    x, y = recipes.c1(300_000)
    y32 = y.astype(np.float32)
    for r in (2, 4, 8, 32):
        a = O.minmaxlttb(x, y32.astype(np.float64), 500, r)
        b = O.minmaxlttb_typed(x, y32, 500, r)
        assert np.array_equal(a, b), r
        pa = O.minmax_preselect(y32, 500, r)
        pb = O.minmax_preselect_typed(y32, 500, r)
        assert np.array_equal(pa, pb)


def _configs():
    p = GOLD / "configs.json"
    if not p.exists():
        pytest.skip("configs.json not generated")
    return json.loads(p.read_text())


def test_oracle_c1_full():
    g = _configs()["C1"]["r4"]["out"]
    x, y = recipes.c1()
    assert O.minmaxlttb(x, y, 1000, 4, threads=O.max_threads()).tolist() == g


def test_oracle_c2_full():
    g = _configs()["C2"]["lttb"]["out"]
    x, y = recipes.c2()
    assert O.lttb(x, y, 2000).tolist() == g


@pytest.mark.slow
def test_oracle_c3_full():
    cfg = _configs()["C3"]
    x, y = recipes.c3()
    for r in recipes.CONFIGS["C3"]["r_ps"]:
        assert O.minmaxlttb_typed(x, y, 2000, r).tolist() == cfg[f"r{r}"]["out"], r


def test_oracle_c4_subset():
    p = GOLD / "c4.json"
    if not p.exists():
        pytest.skip("c4.json not generated")
    g = json.loads(p.read_text())
    x = np.arange(1_000_000, dtype=np.int64)
    for s, out in g["full"].items():
        y = recipes.c4_series(int(s))
        assert O.minmaxlttb_typed(x, y, 1000, 4).tolist() == out
