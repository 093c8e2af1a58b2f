"""Install the unmodified reference (`hebnn`) into baseline/_ref and place its
own test modules beside it (baseline/_ref/hebnn_ref_tests/), so that the
reference's tests can run unmodified against TfheContext on the GPU box
(tests/test_reference_suite.py).  baseline/_ref is git-ignored (not product
source) but travels with the repository snapshot to the GPU box.

Runs only where /root/reference exists (this container); a no-op otherwise.
    python scripts/install_reference.py [--force]
"""

import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference"
TARGET = os.path.join(ROOT, "baseline", "_ref")
TESTS = os.path.join(TARGET, "hebnn_ref_tests")


def install(force=False):
    if not os.path.isdir(REF):
        return False
    if force or not os.path.exists(os.path.join(TARGET, "hebnn", "backend.py")):
        with tempfile.TemporaryDirectory() as tmp:  # the build writes into its source tree
            src = os.path.join(tmp, "pkg")
            shutil.copytree(os.path.join(REF, "pkg"), src, ignore=shutil.ignore_patterns("trainer", "tests"))
            subprocess.run([sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation", "--no-deps",
                            "--find-links", "/opt/wheelhouse", "--target", TARGET, "--upgrade", src], check=True,
                           stdout=subprocess.DEVNULL)
    src_tests = os.path.join(REF, "pkg", "tests")
    os.makedirs(TESTS, exist_ok=True)
    for name in sorted(os.listdir(src_tests)):
        if name.endswith(".py"):
            a, b = os.path.join(src_tests, name), os.path.join(TESTS, name)
            if force or not os.path.exists(b) or os.path.getmtime(a) > os.path.getmtime(b):
                shutil.copy2(a, b)
    return True


if __name__ == "__main__":
    print("installed" if install(force="--force" in sys.argv) else "no /root/reference: nothing to do")
