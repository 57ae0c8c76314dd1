import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
HERE = os.path.dirname(os.path.abspath(__file__))
if HERE not in sys.path:
    sys.path.insert(0, HERE)

GOLDEN = os.path.join(HERE, "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the native library")
    config.addinivalue_line("markers", "slow: large-size GPU checks")
    try:
        from hypothesis import HealthCheck, settings

        settings.register_profile("default", deadline=None, max_examples=60,
                                  suppress_health_check=[HealthCheck.too_slow,
                                                         HealthCheck.filter_too_much])
        settings.load_profile("default")
    except ImportError:  # pragma: no cover
        pass


def err64(original, reconstructed) -> float:
    """float64 max-abs-error (reference conftest.py:14-17)."""
    a = np.asarray(getattr(original, "values", original), dtype=np.float64).ravel()
    b = np.asarray(getattr(reconstructed, "values", reconstructed), dtype=np.float64).ravel()
    return float(np.max(np.abs(a - b)))


class GoldenCases:
    """tests/golden/cases.npz: reference-generated streams (make_golden.py)."""

    def __init__(self):
        self.z = np.load(os.path.join(GOLDEN, "cases.npz"))
        self.meta = json.loads(bytes(self.z["meta"]).decode())

    def __len__(self):
        return len(self.meta)

    def case(self, k):
        m = self.meta[k]
        return (m, self.z[f"x{m['input']}"], bytes(self.z[f"blob{k}"]), self.z[f"recon{k}"])


_golden = None


def golden_cases() -> GoldenCases:
    global _golden
    if _golden is None:
        _golden = GoldenCases()
    return _golden


def golden_digests():
    with open(os.path.join(GOLDEN, "digests.json")) as f:
        return json.load(f)


@pytest.fixture
def rng():
    return np.random.default_rng(0xC0FFEE)


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test selected but no CUDA device is visible")
    return torch
