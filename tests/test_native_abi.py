"""The C-ABI library loads without a GPU and exports every entry point the
header include/hebnn_b200.h declares; host-side calls behave (no compute on
the device is attempted here)."""

import ctypes
import os
import re

import numpy as np
import pytest

from paper_1806_03461_b200 import _native, tfhe

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hebnn_b200.h")


def declared_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(hb_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_binding_table():
    assert set(declared_symbols()) == set(_native.EXPORTED)


def test_library_exports_every_declared_symbol():
    L = _native.lib()
    for name in declared_symbols():
        assert hasattr(L, name), name
        assert ctypes.cast(getattr(L, name), ctypes.c_void_p).value


def test_abi_version_and_params():
    L = _native.lib()
    assert L.hb_abi_version() == 4
    p = _native.default_params()
    assert (p.n, p.N, p.k, p.bg_bits, p.l, p.ks_base_bits, p.ks_t) == (630, 1024, 1, 7, 3, 2, 8)
    assert L.hb_lwe_words(ctypes.byref(p)) == 631
    assert L.hb_ksk_words(ctypes.byref(p)) == 1024 * 8 * 3 * 631
    p.bk_unroll = 1
    assert L.hb_bk_words(ctypes.byref(p)) == 630 * 6 * 2 * 1024
    p.bk_unroll = 2  # key pairs: 3 TGSW per pair
    assert L.hb_bk_words(ctypes.byref(p)) == 315 * 3 * 6 * 2 * 1024


def test_key_pairs_need_even_n():
    p = _native.default_params()
    p.bk_unroll, p.n = 2, 629
    out = np.zeros(4, np.uint32)
    rc = _native.lib().hb_keygen(ctypes.byref(p), 1, _native.u32p(out), _native.u32p(out),
                                 _native.u32p(out), _native.u32p(out), 1)
    assert rc == _native.HB_EINVAL


@pytest.mark.parametrize("n", [640, 750, 1023])
def test_lwe_dimension_beyond_key_switch_columns_is_rejected(n):
    """k_keyswitch writes kKskStride = 640 columns (a_0..a_{n-1}, b): n >= 640 must be
    refused up front instead of returning ciphertexts with unwritten columns."""
    p = _native.default_params()
    assert _native.lib().hb_params_valid(ctypes.byref(p)) == 1
    p.n = n
    assert _native.lib().hb_params_valid(ctypes.byref(p)) == 0
    out = np.zeros(4, np.uint32)
    rc = _native.lib().hb_keygen(ctypes.byref(p), 1, _native.u32p(out), _native.u32p(out),
                                 _native.u32p(out), _native.u32p(out), 1)
    assert rc == _native.HB_EINVAL


def test_invalid_arguments_are_value_errors(keys):
    with pytest.raises(ValueError, match="0 or 1"):
        keys.encrypt(np.array([0, 3], np.uint8), seed=1)
    p = _native.default_params()
    p.N = 2048  # kernels are specialised for N = 1024
    out = np.zeros(4, np.uint32)
    rc = _native.lib().hb_keygen(ctypes.byref(p), 1, _native.u32p(out), _native.u32p(out),
                                 _native.u32p(out), _native.u32p(out), 1)
    assert rc == _native.HB_EINVAL
    with pytest.raises(ValueError):
        _native.check(rc)


def test_gate_record_layout_matches_header():
    assert _native.GATE_DTYPE.itemsize == 24
    assert list(_native.GATE_DTYPE.names) == ["dst", "src_a", "src_b", "src_c", "c0", "alpha", "beta", "kind", "gamma"]


def test_decrypt_host_side(keys):
    bits = np.array([1, 0, 0, 1, 1], np.uint8)
    cts = keys.encrypt(bits, seed=3, stream=2)
    assert np.array_equal(keys.decrypt(cts), bits)
    ph = keys.phase(cts)
    assert np.all((ph > 0) == (bits == 1))


def test_engine_without_gpu_is_a_device_error(keys):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(_native.DeviceError):
        tfhe.Engine(keys, device=0)


def test_gate_dag_rejects_foreign_node_ids():
    """The native gate DAG raises IndexError (never crashes) on ids it does not own."""
    import pytest as _pytest

    d = _native.dag_module().Dag()
    n = d.add_input()
    assert d.gate(0, n << 1, 1) == n << 1  # AND(x, true) = x, no node
    for call in (lambda: d.revive(n + 5), lambda: d.gate(0, (n + 5) << 1, 2), lambda: d.hinc(-1)):
        with _pytest.raises(IndexError):
            call()
