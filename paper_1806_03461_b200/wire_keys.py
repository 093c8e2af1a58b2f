"""Key and ciphertext documents for the client/server split of encrypted
prediction as a service: the client keeps the secret key,
ships evaluation keys (BK, KSK) and encrypted inputs; the server evaluates on
the B200 and returns encrypted outputs.  The reference's wire.py has JSON
documents for models/inputs/reports only (wire.py:143-297) and no ciphertext
format; this adds one, versioned, as .npz (uint32 little-endian arrays) with a
JSON header.
"""

from __future__ import annotations

import ctypes
import json

import numpy as np

from ._native import lib
from .tfhe import KeySet, default_params

FORMAT = "hebnn-b200/tfhe"
VERSION = 2  # 2: params carry bk_unroll (bootstrapping-key layout)
_PARAM_FIELDS = ("n", "N", "k", "bg_bits", "l", "ks_base_bits", "ks_t", "bk_unroll", "lwe_stdev", "bk_stdev")


def _params_doc(p):
    return {f: getattr(p, f) for f in _PARAM_FIELDS}


def _params_from(doc):
    p = default_params()
    for f in _PARAM_FIELDS:
        setattr(p, f, doc[f])
    return p


def _header(kind, params, **extra):
    return json.dumps({"format": FORMAT, "version": VERSION, "kind": kind, "params": _params_doc(params), **extra})


def _check(doc, kind):
    if doc.get("format") != FORMAT or doc.get("version") != VERSION or doc.get("kind") != kind:
        raise ValueError(f"not a {FORMAT} v{VERSION} {kind} document: {doc.get('format')} {doc.get('kind')}")


def save_keys(path, keys, include_secret=False):
    arrays = {"bk": keys.bk, "ksk": keys.ksk}
    if include_secret:
        arrays.update(lwe_key=keys._secret(), trlwe_key=keys.trlwe_key)
    kind = "keyset" if include_secret else "eval_keys"
    np.savez(path, header=np.frombuffer(_header(kind, keys.params, seed=keys.seed).encode(), np.uint8), **arrays)


def _array(z, name, words):
    """A 1-D little-endian uint32 array of exactly `words` elements, else ValueError:
    the engine copies hb_bk_words / hb_ksk_words words from these host buffers."""
    if name not in z.files:
        raise ValueError(f"key document lacks {name!r}")
    a = z[name]
    if a.dtype != np.dtype("<u4") or a.ndim != 1 or a.size != words:
        raise ValueError(f"{name}: expected uint32[{words}], got {a.dtype}{list(a.shape)}")
    return np.ascontiguousarray(a)


def load_keys(path):
    """Load a key document, validating it before any buffer is sized from it: the
    server loads client-supplied files, so params must be ones the kernels support
    and every array must have exactly the length those params imply."""
    with np.load(path, allow_pickle=False) as z:
        doc = json.loads(bytes(z["header"]).decode())
        if doc.get("kind") not in ("keyset", "eval_keys"):
            raise ValueError(f"not a key document: {doc.get('kind')}")
        _check(doc, doc["kind"])
        try:
            p = _params_from(doc["params"])
        except (KeyError, TypeError) as exc:
            raise ValueError(f"bad params in key document: {exc}") from None
        L = lib()
        if not L.hb_params_valid(ctypes.byref(p)):
            raise ValueError(f"key document params not supported by the kernels: {_params_doc(p)}")
        bk = _array(z, "bk", L.hb_bk_words(ctypes.byref(p)))
        ksk = _array(z, "ksk", L.hb_ksk_words(ctypes.byref(p)))
        secret = (None, None)
        if doc["kind"] == "keyset":
            secret = (_array(z, "lwe_key", p.n), _array(z, "trlwe_key", p.k * p.N))
            if (secret[0] > 1).any() or (secret[1] > 1).any():
                raise ValueError("secret keys must be bit vectors")
        ks = KeySet(seed=None, params=p, _arrays=(secret[0], secret[1], bk, ksk))
        ks.seed = doc.get("seed")
        return ks


def save_ciphertexts(path, cts, params, meta=None):
    """cts: uint32 [..., n+1] LWE samples (any leading shape)."""
    cts = np.ascontiguousarray(cts, dtype=np.uint32)
    if cts.shape[-1] != params.n + 1:
        raise ValueError("last axis must be n+1")
    np.savez(path, header=np.frombuffer(_header("ciphertexts", params, meta=meta or {}).encode(), np.uint8), cts=cts)


def load_ciphertexts(path):
    with np.load(path) as z:
        doc = json.loads(bytes(z["header"]).decode())
        _check(doc, "ciphertexts")
        return z["cts"], doc.get("meta", {})
