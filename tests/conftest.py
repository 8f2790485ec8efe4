import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (B200) device and the built libzpir_b200.so")
    config.addinivalue_line("markers", "slow: long-running full-size checks")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


def le_ints(arr):
    a = np.ascontiguousarray(arr, dtype=np.uint8)
    return [int.from_bytes(a[i].tobytes(), "little") for i in range(a.shape[0])]


class Golden:
    def __init__(self, name):
        with open(os.path.join(GOLDEN, f"{name}.json")) as f:
            self.meta = json.load(f)
        self.arr = dict(np.load(os.path.join(GOLDEN, f"{name}.npz")))
        m = self.meta
        self.name = name
        self.lwe = m["lwe"]
        self.d0, self.d1, self.bits = m["d0"], m["d1"], m["paillier_bits"]
        self.p, self.q = int(m["p"], 16), int(m["q"], 16)
        self.m = int(m["m"], 16)
        self.seed = bytes.fromhex(m["client_seed"])
        self.i0 = m["i0"]
        self.cap, self.groups = m["capacity"], m["d1_prime"]
        self.gamma = int(m["gamma"])

    @property
    def db(self):
        if "db" in self.arr:
            return self.arr["db"]
        # tiny: regenerate exactly as the reference bench does (bench.py:167)
        db = np.frombuffer(np.random.default_rng(7).bytes(self.d0 * self.d1),
                           dtype=np.uint8).reshape(self.d0, self.d1)
        return db

    def ints(self, key):
        return le_ints(self.arr[key])

    def params(self, mod):
        """ProtocolParams from either package (`mod` has LweParams/ProtocolParams)."""
        lwe = mod.LweParams(**self.lwe)
        kw = dict(lwe=lwe, d0=self.d0, d1=self.d1, paillier_bits=self.bits)
        if self.meta["scale_regime"] != "quarter_delta":
            kw["scale_regime"] = self.meta["scale_regime"]
        return mod.ProtocolParams(**kw)


# batch scale gamma != 2^32: toy/standard32 (standard regime, general gamma),
# uniform_key (gamma = 2^64), q16 (q = gamma = 2^16)
GAMMA_CASES = ["toy", "uniform_key", "standard32", "q16"]
GPU_CASES = ["desk_reduced", "ragged", "zero_db", "max_db", "tiny"] + GAMMA_CASES
ALL_CASES = GPU_CASES


@pytest.fixture(scope="session")
def golden():
    cache = {}

    def get(name):
        if name not in cache:
            cache[name] = Golden(name)
        return cache[name]
    return get
