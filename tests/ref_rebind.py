"""TEST INFRASTRUCTURE — pytest plugin that runs the reference's own test
modules (baseline/_ref/hebnn_ref_tests/, copied unmodified from
/root/reference/pkg/tests by scripts/install_reference.py) against the drop-in:
every collected module's `SimContext` name, and hebnn.cli's, is rebound to the
context class HB_REF_CTX selects ("gpu": TfheContext on the B200, "plain": the
plaintext stand-in engine for host logic; "-csa" appended: with the opt-in
carry-save popcount) — the rebinding recipe of
INTEGRATION.md §3.  Load with `-p ref_rebind` (tests/ on sys.path)."""

import os
import sys

_HERE = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_HERE)
for _p in (_ROOT, os.path.join(_ROOT, "baseline", "_ref"), _HERE):
    if _p not in sys.path:
        sys.path.insert(0, _p)


def context_class():
    kind = os.environ.get("HB_REF_CTX", "gpu")
    if kind.startswith("plain"):
        from plain_engine import plain_context_class

        base = plain_context_class()
    else:
        from paper_1806_03461_b200.backend import TfheContext as base
    if not kind.endswith("-csa"):
        return base

    class CsaContext(base):  # "plain-csa" / "gpu-csa": the opt-in carry-save popcount (popcount.py)
        def __init__(self, *a, **k):
            k.setdefault("csa_popcount", True)
            super().__init__(*a, **k)

    return CsaContext


def pytest_configure(config):
    import hebnn.cli

    hebnn.cli.SimContext = context_class()


def pytest_collection_modifyitems(session, config, items):
    cls = context_class()
    csa = os.environ.get("HB_REF_CTX", "gpu").endswith("-csa")
    if csa:
        from paper_1806_03461_b200 import popcount
    for item in items:
        mod = getattr(item, "module", None)
        # the test modules imported reduce_tree_sum by name: their direct calls go through the
        # carry-save replacement too (popcount.install() only rebinds the hebnn.* modules)
        if csa and mod is not None and getattr(mod, "reduce_tree_sum", None) is popcount._ORIG:
            mod.reduce_tree_sum = popcount.csa_reduce_tree_sum
        if mod is not None and hasattr(mod, "SimContext") and not getattr(mod, "_hb_rebound", False):
            mod.SimContext = cls
            mod._hb_rebound = True
