"""GPU covering analysis (packing.estimate_covering, packing.py:59-83) against
the reference's own estimates (tests/golden/covering.json, generated from the
reference by tests/golden/make_covering.py): bit-identical rho_hat and
mean_angle."""

import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = json.load(open(os.path.join(HERE, "golden", "covering.json")))


@pytest.mark.parametrize("case", CASES, ids=[f"S{c['S']}_n{c['n_probes']}" for c in CASES])
def test_estimate_covering_matches_reference(cuda, case):
    import paper_2605_27646_b200 as m
    from paper_2605_27646_b200.codebook import SecondaryCodebook

    if case["S"] == 0:
        sec = SecondaryCodebook(np.array([[1.0, 0.0, 0.0, 0.0]]), case["seed"], 0, 0, "K")
    else:
        sec = m.build_secondary(case["seed"], case["layer"], case["head"], case["role"], case["S"])
    est = m.estimate_covering(m.build_joint(sec), case["n_probes"], probe_seed=case["probe_seed"])
    assert est.rho_hat == float.fromhex(case["rho_hat"])
    assert est.mean_angle == float.fromhex(case["mean_angle"])
    assert est.codebook_size == case["codebook_size"] and est.n_probes == case["n_probes"]


def test_estimate_covering_errors(cuda):
    import paper_2605_27646_b200 as m

    with pytest.raises(m.InvalidArgument):
        m.estimate_covering(m.build_joint(m.build_secondary(0, 0, 0, "K", 4)), 0)


def test_covering_cli_matches_reference(cuda, tmp_path):
    """`covering` subcommand (cli.py:136-141,200-210): the same CSV as the
    reference's for --sizes 1,4,16 --seed 2 --probes 20000 --probe-seed 1."""
    from paper_2605_27646_b200 import cli

    out = tmp_path / "cov.csv"
    assert cli.main(["covering", "--sizes", "1,4,16", "--seed", "2", "--probes", "20000",
                     "--probe-seed", "1", "--out", str(out)]) == 0
    want = open(os.path.join(HERE, "golden", "covering_cli.csv")).read()
    assert out.read_text() == want
