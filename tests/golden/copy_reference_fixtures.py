"""Copy the reference's shipped Cancer model (pkg/trainer/out/model.json, the
fixture its CLI tests and SURVEY §8c name) into tests/golden/ so GPU tests can
use it on boxes without /root/reference.  Run once here:
    python tests/golden/copy_reference_fixtures.py
"""

import os
import shutil

SRC = "/root/reference/pkg/trainer/out/model.json"
DST = os.path.join(os.path.dirname(os.path.abspath(__file__)), "cancer_model.json")
shutil.copyfile(SRC, DST)
print("copied", SRC, "->", DST)
