"""Golden covering estimates from the REFERENCE (packing.estimate_covering,
packing.py:59-83) for the GPU re-implementation (paper_2605_27646_b200.covering).

    python oracle/build.py && python tests/golden/make_covering.py
"""

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle", "_ref"))

import hqmq  # noqa: E402  (the reference)
from hqmq.codebook import SecondaryCodebook, build_joint, build_secondary  # noqa: E402
from hqmq.hurwitz import build_primary_codebook  # noqa: E402
from hqmq.kernels import COMPILED_AVAILABLE  # noqa: E402
from hqmq.packing import covering_csv, estimate_covering, fit_covering_rate  # noqa: E402

import numpy as np  # noqa: E402

assert COMPILED_AVAILABLE
assert os.path.realpath(hqmq.__file__).startswith(os.path.join(ROOT, "oracle", "_ref"))

CASES = [  # (S, seed, layer, head, role, n_probes, probe_seed); S = 0: the bare 24-cell
    (0, 0, 0, 0, "K", 5000, 0),
    (16, 0, 0, 0, "K", 20000, 0),
    (64, 3, 5, 2, "V", 50000, 7),
    (256, 0, 79, 7, "K", 8192 + 100, 11),  # crosses the 8192-probe block boundary
]


def main():
    prim = build_primary_codebook()
    out = []
    for (S, seed, layer, head, role, n, ps) in CASES:
        if S == 0:
            sec = SecondaryCodebook(entries=np.array([[1.0, 0.0, 0.0, 0.0]]), seed=seed, layer=0,
                                    head=0, role="K")
        else:
            sec = build_secondary(seed, layer, head, role, S)
        est = estimate_covering(build_joint(prim, sec), n, probe_seed=ps)
        out.append(dict(S=S, seed=seed, layer=layer, head=head, role=role, n_probes=n,
                        probe_seed=ps, rho_hat=est.rho_hat.hex(), mean_angle=est.mean_angle.hex(),
                        codebook_size=est.codebook_size))
    with open(os.path.join(HERE, "covering.json"), "w") as f:
        json.dump(out, f, indent=1)
    # the `covering` CLI table (cli.py:200-210) for sizes 1,4,16 / 20000 probes / seed 2
    fit, est = fit_covering_rate([1, 4, 16], seed=2, n_probes=20000, probe_seed=1)
    with open(os.path.join(HERE, "covering_cli.csv"), "w", newline="") as f:
        covering_csv(est, f)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
