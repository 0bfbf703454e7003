"""Scaling sweeps and benchmark record formats: the host
mirror of run_scaling_sweep / bench_record_json / sweep_csv / time_to_solution
(proj/src/bench.cpp:231-381), checked with the reference's own tests
(proj/tests/test_bench.cpp:142-245) and, where the reference library is built
(oracle/_ref), byte for byte against the reference's output.  CPU only: the
timing model replaces measurement."""
import json
import math

import pytest

import oracle
from paper_2109_04996_b200 import _core

A = math.ldexp(1.0, -20)
B = math.ldexp(1.0, -4)
DIMS = [[8, 8, 8], [12, 12, 12], [16, 16, 16], [20, 20, 20], [21, 21, 21], [22, 22, 22],
        [23, 23, 23], [24, 24, 24], [28, 28, 28], [32, 32, 32], [40, 40, 40], [48, 48, 48]]


def model(a, b):
    return lambda n, P: a * n if P == 1 else a * n / P + b


def test_synthetic_model_efficiency_algebra():
    # test_bench.cpp:142-177
    res = _core.run_scaling_sweep("bp5", 6, DIMS, [1, 2, 4, 8], 20, model=model(A, B))
    rows = res["rows"]
    assert len(rows) == len(DIMS) * 4
    assert all(rows[i]["record"]["n_per_rank"] >= rows[i - 1]["record"]["n_per_rank"]
               for i in range(1, len(rows)))
    for row in rows:
        n, P = row["record"]["n"], row["record"]["P"]
        if P == 1:
            assert row["eta"] == 1.0
        else:
            assert row["eta"] == A * n / (A * n + B * P)
        assert row["T_1"] == A * n
    expected = 4 * B / A
    assert res["summary"]["n08_per_rank"] is not None
    assert abs(res["summary"]["n08_per_rank"] - expected) <= 0.01 * expected
    assert res["summary"]["r_max"] > 0


def test_time_to_solution_identity():
    # test_bench.cpp:180-189
    n08, r08 = 50000.0, 65e6
    t = _core.time_to_solution(1.0, n08 * 512, 0.8, 512, r08 / 0.8)
    assert t == pytest.approx(n08 / r08, rel=1e-12)
    assert 7e-4 <= t <= 9e-4


def test_sweep_requires_serial_baseline():
    with pytest.raises(ValueError, match="must include 1"):
        _core.run_scaling_sweep("bp1", 1, [[2, 2, 2]], [2, 4], 5, model=model(A, B))


def test_measured_multi_rank_needs_a_model():
    with pytest.raises(ValueError, match="one process per GPU"):
        _core.run_scaling_sweep("bp1", 1, [[2, 2, 2]], [1, 2], 5)


def test_record_json_round_trip():
    # test_bench.cpp:198-223
    rec = dict(bp="bp3", p=4, q=6, E=512, n=1030301, P=8, iterations=20,
               seconds=0.12345678901234567)
    rec["dofs_rate"] = rec["n"] * rec["iterations"] / rec["seconds"]
    rec["n_per_rank"] = rec["n"] / rec["P"]
    j = json.loads(_core.bench_record_json(rec))
    assert list(j) == ["bp", "p", "q", "E", "n", "P", "iterations", "seconds", "dofs_rate",
                       "n_per_rank"]
    for k, v in rec.items():
        assert j[k] == v and type(j[k]) is type(v), k


def test_sweep_csv_round_trip():
    # test_bench.cpp:226-245
    a, b = math.ldexp(1.0, -18), math.ldexp(1.0, -5)
    res = _core.run_scaling_sweep("bp2", 3, [[4, 4, 4], [8, 8, 8]], [1, 4], 10, model=model(a, b))
    lines = res["csv"].splitlines()
    assert lines[0] == "bp,p,q,E,n,P,iters,seconds,dofs_rate,n_per_rank,eta" == _core.sweep_csv_header()
    assert len(lines) == 1 + len(res["rows"])
    for line, row in zip(lines[1:], res["rows"]):
        f = line.split(",")
        r = row["record"]
        assert f[0] == r["bp"] and int(f[1]) == r["p"] and int(f[2]) == r["q"]
        assert int(f[3]) == r["E"] and int(f[4]) == r["n"] and int(f[5]) == r["P"]
        assert int(f[6]) == r["iterations"] and float(f[7]) == r["seconds"]
        assert float(f[8]) == r["dofs_rate"] and float(f[9]) == r["n_per_rank"]
        assert float(f[10]) == row["eta"]


def test_summary_of_external_rows_matches_sweep():
    res = _core.run_scaling_sweep("bp5", 6, DIMS[:6], [1, 2, 8], 20, model=model(A, B))
    again = _core.scaling_summary(res["rows"])
    assert again["summary"] == res["summary"] and again["csv"] == res["csv"]


needs_ref = pytest.mark.skipif(not oracle.available("reference"),
                               reason="reference library (oracle/_ref) not built")


@needs_ref
@pytest.mark.parametrize("bp,p,dims,threads,a,b", [
    ("bp5", 6, DIMS, [1, 2, 4, 8], A, B),
    ("bp2", 3, [[4, 4, 4], [8, 8, 8]], [1, 4], math.ldexp(1.0, -18), math.ldexp(1.0, -5)),
    ("bp3", 2, [[3, 2, 2], [5, 5, 4], [9, 9, 9]], [4, 1, 2], 3.3e-9, 1.7e-3),
])
def test_sweep_matches_reference_bytes(bp, p, dims, threads, a, b):
    csv, r_max, n08, C = oracle.sweep_model_reference(bp, p, dims, threads, 20, a, b)
    res = _core.run_scaling_sweep(bp, p, dims, threads, 20, model=model(a, b))
    assert res["csv"] == csv
    s = res["summary"]
    assert s["r_max"] == r_max and s["work_constant"] == C
    assert s["n08_per_rank"] == n08


@needs_ref
def test_record_json_matches_reference():
    rec = dict(bp="bp5", p=7, q=8, E=15625, n=5268024, P=1, iterations=20, seconds=0.0033)
    rec["dofs_rate"] = rec["n"] * rec["iterations"] / rec["seconds"]
    rec["n_per_rank"] = float(rec["n"])
    ours, ref = _core.bench_record_json(rec), oracle.record_json_reference(rec)
    assert json.loads(ours) == json.loads(ref)
    assert list(json.loads(ours)) == list(json.loads(ref))
