"""TEST INFRASTRUCTURE: a plaintext stand-in for the device engine, used only
by CPU tests to check the host-side logic of TfheContext (DAG elision, CSE,
level schedule and the hb_gate record encoding) without a GPU.

Each pool slot holds the *phase* a ciphertext would decrypt to (+-1/8 on the
2^32 torus).  A LIN2 record is executed exactly as the kernel's gate prologue
defines it (c0 + alpha*A + beta*B, then sign -> +-1/8); MUX as the two-
bootstrap CGGI formula.  It is injected by subclassing in tests, never by the
product package.
"""

import functools
import threading

import numpy as np

from paper_1806_03461_b200._native import GATE_HA, GATE_LIN3, GATE_MUX

EIGHTH = 1 << 29


def _sign_to_phase(v):
    v = v.astype(np.uint32).view(np.int32)
    return np.where(v > 0, EIGHTH, -EIGHTH).astype(np.int64)


def _locked(fn):
    """Serialise engine calls like tfhe.Engine does: a background flush runs
    levels while the DAG-building thread grows the pool (reserve replaces the
    array; an unlocked level would write into the old one)."""
    @functools.wraps(fn)
    def wrap(self, *a, **k):
        with self._lock:
            return fn(self, *a, **k)
    return wrap


class PlainEngine:
    def __init__(self, keys):
        self._lock = threading.RLock()
        self.keys = keys
        self.pool = np.zeros(0, np.int64)
        self.records_run = 0
        self.levels_run = 0

    @property
    def capacity(self):
        return self.pool.size

    @_locked
    def reserve(self, slots):
        if slots > self.pool.size:
            self.pool = np.concatenate([self.pool, np.zeros(slots - self.pool.size, np.int64)])

    @_locked
    def upload(self, first, cts):
        ph = self.keys.phase(np.ascontiguousarray(cts, np.uint32)).astype(np.int64)
        self.pool[first:first + len(ph)] = np.where(ph > 0, EIGHTH, -EIGHTH)

    @_locked
    def run_gates(self, recs, lanes=1):
        self.levels_run += 1
        self.records_run += len(recs)
        lane = np.arange(lanes)
        for r in recs:
            A = self.pool[r["src_a"] * lanes + lane]
            B = self.pool[r["src_b"] * lanes + lane]
            if r["kind"] == GATE_HA:
                # one rotation of psi = c0 + alpha A + beta B: S0 = sign(psi), S1 = +1/8 iff
                # psi in [-1/4, 1/4); AND = S0, XOR = gamma (S1 - S0) - gamma/8 (hb_gate HA)
                psi = (int(r["c0"]) + int(r["alpha"]) * A + int(r["beta"]) * B) & 0xFFFFFFFF
                s0 = _sign_to_phase(psi)
                s1 = _sign_to_phase((psi + (1 << 30)) & 0xFFFFFFFF)
                g = int(r["gamma"])
                self.pool[r["src_c"] * lanes + lane] = _sign_to_phase((g * (s1 - s0) - g * EIGHTH) & 0xFFFFFFFF)
                out = s0
            elif r["kind"] == GATE_MUX:
                C = self.pool[r["src_c"] * lanes + lane]
                u1 = _sign_to_phase((-EIGHTH + A + int(r["alpha"]) * B) & 0xFFFFFFFF)
                u2 = _sign_to_phase((-EIGHTH - A + int(r["beta"]) * C) & 0xFFFFFFFF)
                out = _sign_to_phase((EIGHTH + u1 + u2) & 0xFFFFFFFF)
            else:
                v = int(r["c0"]) + int(r["alpha"]) * A + int(r["beta"]) * B
                if r["kind"] == GATE_LIN3:
                    v = v + int(r["gamma"]) * self.pool[r["src_c"] * lanes + lane]
                out = _sign_to_phase(v & 0xFFFFFFFF)
            self.pool[r["dst"] * lanes + lane] = out

    def sync(self):
        pass

    @_locked
    def gather(self, slots):
        # return ciphertexts that decrypt to the stored bits: trivial samples (0, phase)
        n = self.keys.params.n
        out = np.zeros((len(slots), n + 1), np.uint32)
        out[:, n] = (self.pool[np.asarray(slots, np.int64)] & 0xFFFFFFFF).astype(np.uint32)
        return out


def plain_context_class():
    from paper_1806_03461_b200 import backend

    class PlainTfheContext(backend.TfheContext):
        """TfheContext whose flushes run on PlainEngine (host logic only)."""

        def _ensure_engine(self):
            if self._engine is None:
                self._engine = PlainEngine(self.keys)
                self._slots = backend._SlotPool(self._engine)
            return self._engine

    return PlainTfheContext
