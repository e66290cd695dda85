import glob
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


def codec_fixtures():
    out = []
    for path in sorted(glob.glob(os.path.join(GOLDEN, "codec_*.npz"))):
        out.append(os.path.basename(path)[len("codec_"):-4])
    return out


def load_codec_fixture(name):
    z = np.load(os.path.join(GOLDEN, f"codec_{name}.npz"))
    meta = json.loads(str(z["meta"]))
    return meta, {k: z[k] for k in z.files if k != "meta"}


@pytest.fixture(scope="session")
def oracle():
    import hqmq_oracle

    return hqmq_oracle


@pytest.fixture(scope="session")
def cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch.device("cuda", 0)


def adversarial_fixtures():
    return sorted(os.path.basename(p)[len("adv_"):-4]
                  for p in glob.glob(os.path.join(GOLDEN, "adv_*.npz")))


def load_adversarial(name):
    z = np.load(os.path.join(GOLDEN, f"adv_{name}.npz"))
    meta = json.loads(str(z["meta"]))
    return meta, {k: z[k] for k in z.files if k != "meta"}
