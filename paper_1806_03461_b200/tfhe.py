"""Host-side TFHE objects over the C ABI: parameters, key material,
encryption/decryption and the device engine.

These are the real-cryptography counterparts of what the reference's
``SimContext`` does in plaintext (backend.py:171-190): ``KeySet`` is created
where ``SimContext()`` is constructed (cli.py:72), ``encrypt``/``decrypt``
replace ``SimContext.encrypt``/``decrypt``.
"""

from __future__ import annotations

import ctypes
import functools
import threading

import numpy as np

from . import _native
from ._native import GATE_DTYPE, check, lib, u32p

EIGHTH = 1 << 29
MASK32 = 0xFFFFFFFF


def default_params():
    """BASELINE.json configs[0]: n=630, N=1024, k=1, Bg=2^7, l=3, KS 2^2 x 8,
    sigma_lwe = sigma_ks = 2^-15, sigma_bk = 2^-25."""
    return _native.default_params()


class KeySet:
    """Secret keys (LWE, TRLWE) and public evaluation keys (BK, KSK) derived
    deterministically from ``seed`` (ChaCha20 streams)."""

    def __init__(self, seed=0, params=None, threads=0, _arrays=None):
        self.params = params or default_params()
        self.seed = int(seed) if seed is not None else None
        p = self.params
        L = lib()
        if _arrays is not None:  # deserialised (wire_keys.load_keys); secret part may be absent
            self.lwe_key, self.trlwe_key, self.bk, self.ksk = _arrays
            return
        self.lwe_key = np.zeros(p.n, np.uint32)
        self.trlwe_key = np.zeros(p.k * p.N, np.uint32)
        self.bk = np.zeros(L.hb_bk_words(ctypes.byref(p)), np.uint32)
        self.ksk = np.zeros(L.hb_ksk_words(ctypes.byref(p)), np.uint32)
        check(L.hb_keygen(ctypes.byref(p), self.seed, u32p(self.lwe_key), u32p(self.trlwe_key),
                          u32p(self.bk), u32p(self.ksk), threads))

    @property
    def has_secret(self):
        return self.lwe_key is not None

    def public(self):
        """Evaluation keys only (what a server receives): BK + KSK, no secret."""
        return KeySet(seed=None, params=self.params, _arrays=(None, None, self.bk, self.ksk))

    def _secret(self):
        if self.lwe_key is None:
            raise PermissionError("this KeySet holds evaluation keys only (no secret key)")
        return self.lwe_key

    @property
    def lwe_words(self):
        return self.params.n + 1

    def encrypt(self, bits, seed, stream=0, stride=None, first_index=0):
        """Encrypt 0/1 bits -> uint32 [count][stride] LWE samples."""
        bits = np.ascontiguousarray(np.asarray(bits, dtype=np.uint8).reshape(-1))
        stride = stride or self.lwe_words
        out = np.zeros((bits.size, stride), np.uint32)
        check(lib().hb_encrypt(ctypes.byref(self.params), u32p(self._secret()), int(seed), int(stream), int(first_index),
                               bits.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8)), bits.size,
                               u32p(out), stride))
        return out

    def phase(self, cts):
        cts = np.ascontiguousarray(cts, dtype=np.uint32)
        cts2 = cts.reshape(-1, cts.shape[-1])
        out = np.zeros(cts2.shape[0], np.int32)
        check(lib().hb_phase(ctypes.byref(self.params), u32p(self._secret()), u32p(cts2), cts2.shape[0],
                             cts2.shape[1], out.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))))
        return out.reshape(cts.shape[:-1])

    def decrypt(self, cts):
        cts = np.ascontiguousarray(cts, dtype=np.uint32)
        cts2 = cts.reshape(-1, cts.shape[-1])
        out = np.zeros(cts2.shape[0], np.uint8)
        check(lib().hb_decrypt(ctypes.byref(self.params), u32p(self._secret()), u32p(cts2), cts2.shape[0],
                               cts2.shape[1], out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint8))))
        return out.reshape(cts.shape[:-1])


def _locked(fn):
    """Serialise calls into one engine (its stream, staging buffers and pool
    are shared by every context that uses it)."""

    @functools.wraps(fn)
    def wrap(self, *a, **kw):
        with self._lock:
            return fn(self, *a, **kw)

    return wrap


class Engine:
    """One device engine (one CUDA device, one stream) holding the Fourier BK,
    the KSK and a pool of LWE ciphertext slots.  Thread-safe: calls are
    serialised by a per-engine lock."""

    def __init__(self, keys, device=0):
        self._lock = threading.RLock()
        self.keys = keys
        self.params = keys.params
        self._e = ctypes.c_void_p()
        check(lib().hb_engine_create(int(device), ctypes.byref(self.params), u32p(keys.bk), u32p(keys.ksk),
                                     ctypes.byref(self._e)))
        self.device = device

    @_locked
    def close(self):
        if self._e:
            lib().hb_engine_destroy(self._e)
            self._e = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stride(self):
        return lib().hb_pool_stride(self._e)

    @property
    def capacity(self):
        return lib().hb_pool_capacity(self._e)

    @_locked
    def reserve(self, slots):
        check(lib().hb_pool_reserve(self._e, int(slots)))

    @_locked
    def upload(self, first, cts):
        cts = np.ascontiguousarray(cts, dtype=np.uint32)
        check(lib().hb_pool_upload(self._e, int(first), cts.shape[0], u32p(cts), cts.shape[1]))

    @_locked
    def download(self, first, count, out=None):
        """Pool slots [first, first+count) -> host (into `out` [count][>=n+1] if given)."""
        if out is None:
            out = np.zeros((count, self.params.n + 1), np.uint32)
        elif out.dtype != np.uint32 or out.ndim != 2 or out.shape[0] != count or out.shape[1] < self.params.n + 1 \
                or not out.flags.c_contiguous:
            raise ValueError("out must be a C-contiguous uint32 array [count][>= n+1]")
        check(lib().hb_pool_download(self._e, int(first), int(count), u32p(out), out.shape[1]))
        return out

    @_locked
    def upload_async(self, first, cts):
        """Pinned host array -> pool on the copy stream (returns immediately)."""
        check(lib().hb_pool_upload_async(self._e, int(first), cts.shape[0], u32p(cts), cts.shape[1]))

    @_locked
    def download_async(self, first, out):
        """Pool -> pinned host array `out` [count][>=n+1] after all issued levels."""
        check(lib().hb_pool_download_async(self._e, int(first), out.shape[0], u32p(out), out.shape[1]))

    @_locked
    def gather_device(self, slots, dev_ptr, dev_stride):
        """Pool slots -> device buffer at `dev_ptr` (this engine's GPU, rows of
        dev_stride >= n+1 u32 words); synchronous."""
        slots = np.ascontiguousarray(slots, dtype=np.uint32)
        check(lib().hb_pool_gather_device(self._e, u32p(slots), slots.size, ctypes.c_void_p(int(dev_ptr)),
                                          int(dev_stride)))

    @_locked
    def put_device(self, first, count, dev_ptr, dev_stride):
        """Device buffer rows -> pool slots [first, first+count); synchronous."""
        check(lib().hb_pool_put_device(self._e, int(first), int(count), ctypes.c_void_p(int(dev_ptr)),
                                       int(dev_stride)))

    @_locked
    def gather(self, slots):
        slots = np.ascontiguousarray(slots, dtype=np.uint32)
        out = np.zeros((slots.size, self.params.n + 1), np.uint32)
        check(lib().hb_pool_gather(self._e, u32p(slots), slots.size, u32p(out), out.shape[1]))
        return out

    @_locked
    def run_gates(self, gates, lanes=1):
        """gates: numpy array of GATE_DTYPE records (one level)."""
        gates = np.ascontiguousarray(gates, dtype=GATE_DTYPE)
        check(lib().hb_run_gates(self._e, gates.ctypes.data_as(ctypes.c_void_p), gates.shape[0], int(lanes)))

    def sync(self):
        """Wait for the engine's streams.  Not under the engine lock: hb_sync only
        synchronises streams, so a background flush waiting here does not block
        other threads' calls (pool growth, uploads, the next level)."""
        check(lib().hb_sync(self._e))

    @_locked
    def last_timing(self):
        a, b = ctypes.c_float(), ctypes.c_float()
        check(lib().hb_last_timing(self._e, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    @_locked
    def counters(self):
        a, b, c = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
        check(lib().hb_counters(self._e, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return {"blind_rotations": a.value, "key_switches": b.value, "kernel_launches": c.value}

    @_locked
    def flush_l2(self, nbytes=0):
        check(lib().hb_flush_l2(self._e, int(nbytes)))

    @_locked
    def measure_fp64_peak(self):
        v = ctypes.c_double()
        check(lib().hb_measure_fp64_peak(self._e, ctypes.byref(v)))
        return v.value

    # ---- stage entry points (parity) ----
    @_locked
    def debug_blind_rotate(self, lwe, mu=EIGHTH, iters=-1):
        out = np.zeros(2 * self.params.N, np.uint32)
        check(lib().hb_debug_blind_rotate(self._e, u32p(np.ascontiguousarray(lwe, np.uint32)), mu, iters, u32p(out)))
        return out

    @_locked
    def debug_bootstrap_wo_ks(self, lin):
        lin = np.ascontiguousarray(lin, dtype=np.uint32).reshape(-1, self.params.n + 1)
        out = np.zeros((lin.shape[0], self.params.N + 1), np.uint32)
        check(lib().hb_debug_bootstrap_wo_ks(self._e, u32p(lin), lin.shape[0], u32p(out)))
        return out

    @_locked
    def debug_keyswitch(self, big):
        big = np.ascontiguousarray(big, dtype=np.uint32).reshape(-1, self.params.N + 1)
        out = np.zeros((big.shape[0], self.params.n + 1), np.uint32)
        check(lib().hb_debug_keyswitch(self._e, u32p(big), big.shape[0], u32p(out)))
        return out

    @_locked
    def debug_fourier(self, polys=None, count=None, which=0):
        if which == 1:
            out = np.zeros((count, self.params.N // 2, 2), np.float64)
            dummy = np.zeros(1, np.uint32)
            check(lib().hb_debug_fourier(self._e, u32p(dummy), count, out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 1))
        else:
            polys = np.ascontiguousarray(polys, dtype=np.uint32).reshape(-1, self.params.N)
            out = np.zeros((polys.shape[0], self.params.N // 2, 2), np.float64)
            check(lib().hb_debug_fourier(self._e, u32p(polys), polys.shape[0],
                                         out.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 0))
        return out[..., 0] + 1j * out[..., 1]

    @_locked
    def debug_fft_margin(self):
        v = ctypes.c_double()
        check(lib().hb_debug_fft_margin(self._e, ctypes.byref(v)))
        return v.value


def gate_records(n):
    return np.zeros(n, dtype=GATE_DTYPE)


# (c0, alpha, beta) of each CGGI boolean gate over the +-1/8 encoding
GATE_LIN = {
    "AND": ((-EIGHTH) & MASK32, 1, 1),
    "OR": (EIGHTH, 1, 1),
    "XOR": (2 * EIGHTH, 2, 2),
    "XNOR": ((-2 * EIGHTH) & MASK32, -2, -2),
    "NAND": (EIGHTH, -1, -1),
    "NOR": ((-EIGHTH) & MASK32, -1, -1),
}
