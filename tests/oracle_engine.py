"""TEST INFRASTRUCTURE: runs TfheContext flushes on the exact CPU oracle
(oracle/tfhe_oracle.c, pthreads) instead of the B200, so the reference's
decrypted-bit semantics can be replayed on *real* CGGI ciphertexts on a
machine without a GPU.  Injected by subclassing in tests only.
"""

import os

import numpy as np

from oracle import oracle as O


class OracleEngine:
    def __init__(self, keys):
        self.keys = keys
        self.p = O.default_params()
        self.p.bk_unroll = keys.params.bk_unroll
        ok = O.Keys(self.p, keys.seed)
        assert np.array_equal(ok.lwe_key, keys.lwe_key), "oracle and product keys differ"
        self.ctx = O.Context(self.p, ok)
        self.words = self.p.n + 1
        self.pool = np.zeros((0, self.words), np.uint32)
        self.threads = os.cpu_count() or 1
        self.bootstraps = 0

    @property
    def capacity(self):
        return self.pool.shape[0]

    def reserve(self, slots):
        if slots > self.pool.shape[0]:
            grow = np.zeros((slots - self.pool.shape[0], self.words), np.uint32)
            self.pool = np.ascontiguousarray(np.concatenate([self.pool, grow]))

    def upload(self, first, cts):
        cts = np.asarray(cts, np.uint32).reshape(-1, self.words)
        self.pool[first:first + cts.shape[0]] = cts

    def run_gates(self, recs, lanes=1):
        recs = np.asarray(recs)
        if lanes != 1:  # expand lanes into per-lane records on physical slots
            out = np.repeat(recs, lanes)
            lane = np.tile(np.arange(lanes, dtype=np.uint32), recs.size)
            for f in ("dst", "src_a", "src_b", "src_c"):
                out[f] = out[f] * lanes + lane
            recs = out
        self.bootstraps += int(recs.size + np.count_nonzero(recs["kind"] == 1) - np.count_nonzero(recs["kind"] == 3))
        self.ctx.run_gates(recs, self.pool, threads=self.threads)

    def sync(self):
        pass

    def gather(self, slots):
        return self.pool[np.asarray(slots, np.int64)].copy()


def oracle_context_class():
    from paper_1806_03461_b200 import backend

    class OracleTfheContext(backend.TfheContext):
        """TfheContext whose flushes run on the CPU oracle (exact CGGI)."""

        def _ensure_engine(self):
            if self._engine is None:
                self._engine = OracleEngine(self.keys)
                self._slots = backend._SlotPool(self._engine)
            return self._engine

    return OracleTfheContext
