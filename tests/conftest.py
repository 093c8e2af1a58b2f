import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
for p in (ROOT, REF):
    if p not in sys.path:
        sys.path.insert(0, p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (run via gpurun)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def cuda_available():
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:  # pragma: no cover
        return False


@pytest.fixture(scope="session")
def keys():
    from paper_1806_03461_b200 import tfhe

    return tfhe.KeySet(seed=42)


@pytest.fixture(scope="session")
def okeys():
    from oracle import oracle as O

    return O.Keys(O.default_params(), 42)


@pytest.fixture(scope="session")
def octx(okeys):
    from oracle import oracle as O

    return O.Context(O.default_params(), okeys)


@pytest.fixture(scope="session")
def engine(keys):
    from paper_1806_03461_b200 import tfhe

    eng = tfhe.Engine(keys, device=0)
    yield eng
    eng.close()
