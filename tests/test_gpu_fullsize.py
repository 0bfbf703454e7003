"""Parity at BASELINE.json's full sizes — the configurations bench.py and the
sweeps time, against the reference itself
(oracle/_ref, the unmodified hexfem compiled from its sources, run on all
host cores).  Bars: apply rel_max_diff <= 1e-12; the bench step's 20 fixed
CG iterations: residual history and iterate within 1e-10 (FMA / RED
rounding differences are ~1e-15 per apply).

Each case builds the reference problem on the host (seconds) — these are the
slowest GPU tests."""
import os

import numpy as np
import pytest

import oracle
from gpu_common import op_from_oracle
from paper_2109_04996_b200 import capi

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not oracle.available("reference"),
                                 reason="oracle/_ref not built (make -C oracle ref)")]

THREADS = os.cpu_count() or 1
APPLY_TOL = 1e-12


@pytest.fixture(scope="module")
def ctx():
    c = capi.Context(0)
    yield c
    c.close()


def ref_problem(bp, p, d):
    return oracle.setup(bp, p, (d, d, d), "sine", threads=THREADS, impl="reference")


def test_c3_bp5_p7_25cubed_apply_and_bench_step(ctx):
    """C3 = the bench workload: BP5 p=7 25^3 (5.27 M DOFs), DMMA kernel with
    ~26 elements per CTA."""
    ref = ref_problem("bp5", 7, 25)
    op = op_from_oracle(ctx, ref)
    assert op.structured
    for seed in (99, 64):
        x = oracle.seeded_uniform(ref.size, seed)
        assert oracle.rel_max_diff(ref.apply(x), op.apply(x)) <= APPLY_TOL
    d = ref.diagonal()
    assert np.array_equal(op.diagonal(), d)
    x, rep = op.pcg(ref.rhs, d, tol=1e-8, fixed_iterations=20)
    xr, rrep = ref.solve(tol=1e-8, fixed_iterations=20)
    assert rep["iterations"] == rrep["iterations"] == 20
    assert oracle.rel_max_diff(rrep["residual_history"], rep["residual_history"]) <= 1e-10
    assert oracle.rel_max_diff(xr, x) <= 1e-10


def test_c2_bp3_p7_31cubed_apply(ctx):
    """C2: BP3 p=7 q=9, 31^3 (10.08 M DOFs), line kernel with staged factors."""
    ref = ref_problem("bp3", 7, 31)
    op = op_from_oracle(ctx, ref)
    x = oracle.seeded_uniform(ref.size, 99)
    assert oracle.rel_max_diff(ref.apply(x), op.apply(x)) <= APPLY_TOL


@pytest.mark.parametrize("p,d", [(5, 48), (6, 40), (7, 34), (8, 30)],
                         ids=["p5-pencil", "p6-padded-dmma", "p7-dmma", "p8-pencil"])
def test_c4_bp6_apply(ctx, p, d):
    """C4: BP6 (3 components), ~41 M DOFs, one order per three-component kernel."""
    ref = ref_problem("bp6", p, d)
    op = op_from_oracle(ctx, ref)
    x = oracle.seeded_uniform(ref.size, 64)
    assert oracle.rel_max_diff(ref.apply(x), op.apply(x)) <= APPLY_TOL
