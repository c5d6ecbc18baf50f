import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: long-running parity case")


class Golden:
    """A fixture written by oracle/make_golden.py from the reference's own outputs."""

    def __init__(self, name):
        self.name = name
        self.z = np.load(GOLDEN / f"{name}.npz")
        self.meta = json.loads(bytes(self.z["meta_json"]).decode())
        self.dims = tuple(self.meta["dims"])
        self.n = int(np.prod(self.dims))

    def __getitem__(self, k):
        return self.z[k]

    def __contains__(self, k):
        return k in self.z.files

    @property
    def family(self):
        return {"haar": 0, "daubechies": 1, "symmlet": 2}[self.meta["family"]]

    def generator_list(self):
        from paper_1512_08401_b200 import waveblur as W
        return W.GeneratorList(self.dims, self.meta["J"], W.FilterFamily(self.family), self.meta["order"],
                               self["gen_block"].astype(np.uint32), self["gen_index"].astype(np.uint32),
                               self["gen_count"].astype(np.uint64), self["gen_value"])

    def operator(self):
        from paper_1512_08401_b200 import waveblur as W
        return W.theta_from_generators(self.generator_list())

    def weights(self):
        from paper_1512_08401_b200 import waveblur as W
        return W.scale_weights(W.make_layout(self.dims, self.meta["J"]))


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = Golden(name)
        return cache[name]
    return get


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
