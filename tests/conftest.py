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


# Default key layout (bk_unroll 2, key pairs) and, suffixed 1, the CGGI layout
# (bk_unroll 1, one TGSW per key bit); both are product paths with their own
# oracle restatement and golden vectors.

def oracle_params(unroll=None):
    from oracle import oracle as O

    p = O.default_params()
    if unroll is not None:
        p.bk_unroll = unroll
    return p


def product_params(unroll=None):
    from paper_1806_03461_b200 import tfhe

    p = tfhe.default_params()
    if unroll is not None:
        p.bk_unroll = unroll
    return p


@pytest.fixture(scope="session")
def keys():
    from paper_1806_03461_b200 import tfhe

    return tfhe.KeySet(seed=42)


@pytest.fixture(scope="session")
def okeys():
    from oracle import oracle as O

    return O.Keys(oracle_params(), 42)


@pytest.fixture(scope="session")
def octx(okeys):
    from oracle import oracle as O

    return O.Context(oracle_params(), okeys)


@pytest.fixture(scope="session")
def engine(keys):
    from paper_1806_03461_b200 import tfhe

    eng = tfhe.Engine(keys, device=0)
    yield eng
    eng.close()


@pytest.fixture(scope="session")
def keys1():
    from paper_1806_03461_b200 import tfhe

    return tfhe.KeySet(seed=42, params=product_params(1))


@pytest.fixture(scope="session")
def okeys1():
    from oracle import oracle as O

    return O.Keys(oracle_params(1), 42)


@pytest.fixture(scope="session")
def octx1(okeys1):
    from oracle import oracle as O

    return O.Context(oracle_params(1), okeys1)


@pytest.fixture(scope="session")
def engine1(keys1):
    from paper_1806_03461_b200 import tfhe

    eng = tfhe.Engine(keys1, device=0)
    yield eng
    eng.close()
