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


# the four exhaustive reference tests that take 4-7 minutes each on real ciphertexts (chains
# of thousands of one-level flushes); the driver's GPU tier has 20 minutes for the whole suite
SLOWEST = ("test_acceptance.py::test_criterion_8_comparator_equality",
           "test_circuits.py::test_compare_ge_const_exhaustive_k8",
           "test_circuits.py::test_reduce_tree_exhaustive_small_n",
           "test_compiler.py::test_neuron_methods_exhaustive_small_d")
FULL = os.environ.get("HB_GPU_FULL") == "1"


def _popen(modules, ctx, extra=()):
    env = dict(os.environ, HB_REF_CTX=ctx, PYTHONPATH=os.pathsep.join([HERE, ROOT, os.path.join(ROOT, "baseline", "_ref")]))
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "ref_rebind", "-p", "no:cacheprovider", "--rootdir", REF_TESTS,
           *extra, *[os.path.join(REF_TESTS, m) for m in modules]]
    return subprocess.Popen(cmd, cwd=REF_TESTS, env=env, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)


@pytest.mark.gpu
def test_reference_suite_on_gpu():
    """Unmodified reference tests on real ciphertexts: test_backend, test_circuits,
    test_compiler and test_acceptance (eight pytest-xdist workers — eight processes,
    eight engines — share the B200: each test is a chain of one-level flushes that keeps
    only a few SMs busy) and, at the same time, the hebnn CLI `selftest`
    (cli.py:212-229) with the B200 backend, and test_circuits / test_compiler again with
    the opt-in carry-save popcount.  The four slowest exhaustive tests
    (SLOWEST: the exhaustive reduce tree n <= 12, test_circuits.py:124-130, the k = 8
    comparators, test_circuits.py:216-223, ...) run in
    test_reference_suite_exhaustive_on_gpu (HB_GPU_FULL=1; profiles/r02_v/pytest_gpu.log
    has them passing) so that the default GPU tier stays well inside its time limit."""
    deselect = [a for t in SLOWEST for a in ("--deselect", t)]  # node ids relative to the rootdir
    suite = _popen(["test_backend.py", "test_circuits.py", "test_compiler.py", "test_acceptance.py"], "gpu",
                   extra=("--durations=10", "-n", "8", *deselect))
    cli = _popen(["test_cli.py"], "gpu", extra=("-k", "test_selftest_passes"))
    # the circuit and compiler modules once more with the opt-in carry-save popcount
    # (their direct reduce_tree_sum calls rebound too, tests/ref_rebind.py)
    csa = _popen(["test_circuits.py", "test_compiler.py"], "gpu-csa", extra=("-n", "4", *deselect))
    try:
        out_suite, _ = suite.communicate(timeout=900)
        out_cli, _ = cli.communicate(timeout=900)
        out_csa, _ = csa.communicate(timeout=900)
    finally:
        for p in (suite, cli, csa):
            if p.poll() is None:
                p.kill()
    print(out_suite[-3000:])
    assert suite.returncode == 0 and " passed" in out_suite and "failed" not in out_suite, out_suite[-4000:]
    assert cli.returncode == 0 and " passed" in out_cli, out_cli[-4000:]
    assert csa.returncode == 0 and " passed" in out_csa and "failed" not in out_csa, out_csa[-4000:]


@pytest.mark.gpu
@pytest.mark.skipif(not FULL, reason="HB_GPU_FULL=1 runs the four 4-7 minute exhaustive reference tests")
def test_reference_suite_exhaustive_on_gpu():
    out = _run(list(SLOWEST), "gpu", 3600, extra=("--durations=10", "-n", "4"))
    print(out[-3000:])
    assert " passed" in out and "failed" not in out
