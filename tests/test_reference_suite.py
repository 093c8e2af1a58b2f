"""The reference's own tests, unmodified, against the drop-in:
pytest runs baseline/_ref/hebnn_ref_tests/{test_backend,test_circuits,
test_compiler,...}.py (copies of /root/reference/pkg/tests made by
scripts/install_reference.py) with `SimContext` rebound by tests/ref_rebind.py.

CPU: the host logic (DAG, elision, fusion, streaming, stats, scopes, errors)
on the plaintext stand-in engine.  GPU: real CGGI ciphertexts on the B200, plus
the acceptance criteria and the CLI (its `selftest` included)."""

import os
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
REF_TESTS = os.path.join(ROOT, "baseline", "_ref", "hebnn_ref_tests")

pytestmark = pytest.mark.skipif(not os.path.isdir(REF_TESTS),
                                reason="reference tests not installed (python scripts/install_reference.py)")


def _run(modules, ctx, timeout, extra=()):
    env = dict(os.environ, HB_REF_CTX=ctx, PYTHONPATH=os.pathsep.join([HERE, ROOT, os.path.join(ROOT, "baseline", "_ref")]))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "ref_rebind", "-p", "no:cacheprovider", "--rootdir", REF_TESTS,
           *extra, *[os.path.join(REF_TESTS, m) for m in modules]]
    r = subprocess.run(cmd, cwd=REF_TESTS, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, (r.stdout[-4000:], r.stderr[-2000:])
    return r.stdout


def test_reference_suite_on_plain_engine():
    out = _run(["test_backend.py", "test_circuits.py", "test_compiler.py"], "plain", 900)
    assert " passed" in out and "failed" not in out


def test_reference_suite_on_plain_engine_with_csa_popcount():
    """The same unmodified modules with the opt-in carry-save popcount: the
    reference's own gate-count, level and value assertions on reduce_tree_sum
    and the compiler hold (popcount.py charges the reference's counts)."""
    out = _run(["test_backend.py", "test_circuits.py", "test_compiler.py"], "plain-csa", 900)
    assert " passed" in out and "failed" not in out


@pytest.mark.gpu
def test_reference_suite_on_gpu():
    """Unmodified reference tests on real ciphertexts, all of them, including the
    exhaustive reduce tree (n <= 12, test_circuits.py:124-130) and k = 8
    comparators (test_circuits.py:216-223) the round-1 GPU tier had reduced.
    Each test is a chain of thousands of one-level flushes (sequential bootstrap
    latency, a few SMs busy), so eight pytest-xdist workers — eight processes,
    eight engines — share the B200."""
    out = _run(["test_backend.py", "test_circuits.py", "test_compiler.py", "test_acceptance.py"], "gpu", 3600,
               extra=("--durations=10", "-n", "8"))
    print(out[-3000:])
    assert " passed" in out and "failed" not in out


@pytest.mark.gpu
def test_reference_cli_selftest_on_gpu():
    """hebnn CLI `selftest` (cli.py:212-229) with the B200 backend."""
    out = _run(["test_cli.py"], "gpu", 1800, extra=("-k", "test_selftest_passes"))
    assert " passed" in out
