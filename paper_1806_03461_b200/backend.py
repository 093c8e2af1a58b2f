"""`TfheContext`: the reference's `GateBackend` (backend.py:116-150) on real
CGGI/TFHE ciphertexts, executed on a B200.

Drop-in contract, reproduced from `SimContext`
(backend.py:161-257):

* `encrypt`/`trivial_const` raise ValueError unless b in {0, 1} (178-186);
* gate methods return `CipherBit` handles whose `level` follows the ASAP rule
  (207, 235), whose `trivial_value` is set only for trivial constants, and
  whose `.context` is this context;
* `GateStats` counting (`_record`, 199-203), nested scopes (241-249),
  `gate_count`/`scope_depth` (251-257) and the lock that makes concurrent gate
  issue race-free (174, 200) are identical;
* `ContextMismatchError` for foreign handles (194-197), `ScopeError` on scope
  underflow; device failures raise `DeviceError` (never ValueError);
* NOT is free unless `hebnn.backend.NOT_IS_FREE` is False (223-228); a MUX on
  a trivial selector is free and returns the very same handle (232-234).

Execution is lazy: gates append nodes to a DAG; `decrypt` (the only flush point
of the reference API) runs every pending node on the GPU one level at a time
(the level histogram is the batch schedule).  While building the
DAG, gates whose result is already determined are not bootstrapped (trivial
inputs, repeated inputs, common subexpressions, MUX with trivial data inputs);
a full adder's OR(AND(a,b), AND(XOR(a,b),c)) becomes one 3-input majority
bootstrap and XOR(XOR(a,b),c) one 3-input XOR bootstrap (hb_gate LIN3), and a
flush executes only the pending gates that a live handle still reaches (the
rest stay in the DAG, dormant, and run if they are ever needed again).  The
counted `GateStats` are unaffected and decrypted values are identical
(SURVEY.md §8 f2).  With ``lanes = B`` every handle carries B independent
ciphertexts that share one DAG.
"""

from __future__ import annotations

import os
import threading
import time
import weakref

import numpy as np

try:  # the reference's own plugin interface (backend.py:23-150): a hard dependency of the drop-in
    from hebnn import backend as _ref_backend
    from hebnn.backend import AND, MUX, OR, XNOR, XOR, CipherBit, ContextMismatchError, GateBackend, GateStats, ScopeError
except ImportError as _exc:  # pragma: no cover
    raise ImportError("paper_1806_03461_b200.backend implements hebnn.backend.GateBackend: install the reference "
                      "package (pip install --target baseline/_ref /root/reference/pkg) or put it on sys.path") from _exc

from ._native import GATE_DTYPE, GATE_HA, GATE_LIN2, GATE_LIN3, GATE_MUX, dag_module
from .tfhe import EIGHTH, MASK32, Engine, KeySet

# node opcodes of the native gate DAG (csrc/hb_dag.cpp): node 0 is the constant 0
# (ref 0 = false, ref 1 = true); refs are (node << 1) | NOT flag
_DAG = dag_module()
_OP_INPUT = _DAG.OP_INPUT
_OP_AND = _DAG.OP_AND
_OP_XOR = _DAG.OP_XOR
_OP_MUX = _DAG.OP_MUX
_OP_MAJ = _DAG.OP_MAJ
_OP_XOR3 = _DAG.OP_XOR3
_KIND = {AND: 0, OR: 1, XOR: 2, XNOR: 3}  # Dag.gate kinds

_C_AND = (-EIGHTH) & MASK32
_C_XOR = 2 * EIGHTH


class DeviceError(RuntimeError):
    """Raised when the B200 engine cannot run (no device, CUDA failure).  The
    gates of the failed flush count as executed, so a context that raised it
    must not be decrypted from again (create a new one)."""


class _Bit(CipherBit):
    """`CipherBit` that tells its context when it dies, so a flush can skip
    gates no live handle reaches (the handle contract is the reference's)."""

    __slots__ = ()

    def __del__(self):
        try:
            self._ctx._dag.hdec(self._value >> 1)
        except Exception:  # interpreter shutdown
            pass


# ---------------------------------------------------------------------------
# shared engines and slot allocation
# ---------------------------------------------------------------------------

_KEY_CACHE = {}
_ENGINE_CACHE = {}
_CACHE_LOCK = threading.Lock()
_CONTEXT_SERIAL = 0


def shared_keys(seed):
    """Key sets are deterministic in the seed; contexts with equal seeds share
    one (keygen costs ~1 s on the host)."""
    with _CACHE_LOCK:
        ks = _KEY_CACHE.get(seed)
        if ks is None:
            ks = _KEY_CACHE[seed] = KeySet(seed=seed)
        return ks


class _SlotPool:
    """First-fit allocator of physical pool slots on one engine."""

    def __init__(self, engine):
        self.engine = engine
        self.top = 0
        self.free = []  # (base, size)
        self.lock = threading.Lock()

    def alloc(self, size, align=1):
        with self.lock:
            for i, (b, s) in enumerate(self.free):
                ab = -(-b // align) * align
                if ab + size <= b + s:
                    del self.free[i]
                    if ab > b:
                        self.free.append((b, ab - b))
                    if ab + size < b + s:
                        self.free.append((ab + size, b + s - ab - size))
                    return ab
            ab = -(-self.top // align) * align
            if ab > self.top:
                self.free.append((self.top, ab - self.top))
            self.top = ab + size
            if self.top > self.engine.capacity:
                self.engine.reserve(max(self.top, int(self.engine.capacity * 1.5) + 1024))
            return ab

    def release(self, base, size):
        with self.lock:
            self.free.append((base, size))


def shared_engine(keys, device):
    key = (id(keys.bk), device)
    with _CACHE_LOCK:
        ent = _ENGINE_CACHE.get(key)
        if ent is None:
            try:
                eng = Engine(keys, device=device)
            except (RuntimeError, OSError) as exc:
                raise DeviceError(f"cannot create the B200 engine on device {device}: {exc}") from exc
            ent = _ENGINE_CACHE[key] = (eng, _SlotPool(eng))
        return ent


def _release_chunks(pool, *chunk_lists):
    for chunks in chunk_lists:
        for base, size in chunks:
            pool.release(base, size)


# ---------------------------------------------------------------------------
# the context
# ---------------------------------------------------------------------------


class TfheContext(GateBackend):
    """CGGI/TFHE gate-bootstrapping backend on a B200 (see module docstring).

    Parameters
    ----------
    seed:     key seed (keys are deterministic in it; equal seeds share keys)
    device:   CUDA device ordinal of the engine
    lanes:    independent ciphertexts per handle (one DAG, B executions)
    enc_seed: seed of the encryption randomness (defaults to ``seed``)
    enc_stream: ChaCha stream id of this context's encryptions (defaults to a
              per-process creation counter, so runs are reproducible)
    keys:     an explicit `KeySet` (overrides ``seed``)
    stream_at: pending gates that start a background flush while the DAG is
              still being built (0 disables; flush points are unchanged)
    fuse_half_adders: an XOR and an AND/OR of the same two nodes in one flush
              run as one HA record: one blind rotation extracted twice (the
              AND at index 0, the XOR from the difference of the index-N/2 and
              index-0 extractions), two key switches.
    stream_min_width: bootstraps a level needs in a background flush; narrower
              levels (and the gates that depend on them) stay pending and
              merge with later gates of the same level (the final flush runs
              everything).  A narrow launch costs about as much as a full
              wave, so this keeps streamed launches wide.  0 disables.
    csa_popcount: opt-in (default: environment HEBNN_B200_CSA_POPCOUNT, else off
              = the pure drop-in).  Rebinds the
              reference's `reduce_tree_sum` (popcount.py) so that popcounts of
              this context's bits are built as carry-save compressor networks
              (~2n instead of ~3n bootstraps for n bits); decrypted words and
              counted `GateStats` are unchanged.
    """

    _CHUNK = 4096  # logical slots reserved at a time

    def __init__(self, seed=0, device=0, lanes=1, enc_seed=None, keys=None, enc_stream=None, stream_at=16384,
                 stream_min_width=592, fuse_half_adders=True, csa_popcount=None):
        if lanes < 1:
            raise ValueError("lanes must be >= 1")
        self.global_stats = GateStats(label="global")
        self._scopes = []
        self._lock = threading.RLock()
        self.keys = keys if keys is not None else shared_keys(seed)
        self.params = self.keys.params
        self.device = device
        self.lanes = int(lanes)
        self.enc_seed = seed if enc_seed is None else enc_seed
        self._enc_count = 0
        global _CONTEXT_SERIAL
        with _CACHE_LOCK:
            _CONTEXT_SERIAL += 1
            serial = _CONTEXT_SERIAL
        self.enc_stream = (serial if enc_stream is None else int(enc_stream)) & 0xFFFFF
        # gate DAG (native, csrc/hb_dag.cpp): node store, elision, CSE, full-adder
        # fusion, live-handle counts; logical pool slot of node n is n - 1
        self._dag = _DAG.Dag()
        self._inputs = {}      # node id -> host ciphertexts [lanes][n+1] not yet uploaded
        self._engine = None
        self._slots = None
        self._history = []     # every executed (level, records) batch, in order (f1 replay)
        self._chunks = []
        self._sched_chunks = []  # pool chunks of compiled-schedule runs (run_schedule)
        self._finalizer = None
        self.stream_at = int(stream_at)  # pending gates that start a background flush (0: off)
        self.stream_min_width = int(stream_min_width)
        self.fuse_half_adders = bool(fuse_half_adders)
        # opt-in: the compiler's popcounts (hebnn.circuits.reduce_tree_sum) run as carry-save
        # compressor networks built in the DAG (popcount.py); counted stats stay the reference's
        if csa_popcount is None:
            csa_popcount = os.environ.get("HEBNN_B200_CSA_POPCOUNT", "0") not in ("", "0")
        self.csa_popcount = bool(csa_popcount)
        # shared first stage of the carry-save popcounts: leaf ordinals per block (0: none)
        self.csa_block = int(os.environ.get("HEBNN_B200_CSA_BLOCK", "7"))
        if self.csa_popcount:
            from . import popcount

            popcount.install()
        # gates between two streaming checks (a countdown instead of a native call per gate)
        self._tick_every = max(1, min(256, self.stream_at // 8))
        self._tick = self._tick_every
        self._bg = None
        self._bg_error = []
        # execution statistics
        self.exec_stats = {"bootstraps": 0, "gates": 0, "levels": 0, "device_ms": 0.0, "flushes": 0,
                           "flush_s": 0.0}

    # -- engine / slots ------------------------------------------------------

    def _ensure_engine(self):
        if self._engine is None:
            self._engine, self._slots = shared_engine(self.keys, self.device)
            self._finalizer = weakref.finalize(self, _release_chunks, self._slots, self._chunks, self._sched_chunks)
        return self._engine


    def _map_slots(self, logical, chunks=None, count=None):
        """Logical slots -> engine record slots (chunks of the shared pool are
        reserved on demand, aligned to `lanes` so slot * lanes + lane is the
        physical pool index).  `chunks`/`count`: another chunk list (compiled
        schedules) covering `count` logical slots."""
        self._ensure_engine()
        if chunks is None:
            chunks, count = self._chunks, self._dag.size()
        need = (max(count, 1) - 1) // self._CHUNK + 1
        while len(chunks) < need:
            base = self._slots.alloc(self._CHUNK * self.lanes, align=self.lanes)
            chunks.append((base, self._CHUNK * self.lanes))
        bases = np.array([b // self.lanes for b, _ in chunks], dtype=np.int64)
        logical = np.asarray(logical, dtype=np.int64)
        return bases[logical // self._CHUNK] + logical % self._CHUNK

    def _unmap_slots(self, phys):
        """Inverse of _map_slots over this context's chunks; record slots outside
        them (the unused src_c of two-input records) map to logical 0."""
        bases = np.array([b // self.lanes for b, _ in self._chunks], dtype=np.int64)
        order = np.argsort(bases)
        phys = np.asarray(phys, dtype=np.int64)
        k = np.searchsorted(bases[order], phys, side="right") - 1
        ok = k >= 0
        ci = order[np.maximum(k, 0)]
        off = phys - bases[ci]
        ok &= (off >= 0) & (off < self._CHUNK)
        return np.where(ok, ci * self._CHUNK + off, 0)

    # -- checks / stats (SimContext._check/_record, backend.py:194-203) --------

    def _check(self, *bits):
        for c in bits:
            if not isinstance(c, CipherBit) or c._ctx is not self:
                raise ContextMismatchError("bit handle does not belong to this context")

    def _record(self, kind, level):
        self.global_stats.record(kind, level)
        for scope in self._scopes:
            scope.record(kind, level)

    # -- bit creation ----------------------------------------------------------

    def _bit(self, r, level, trivial=None):
        """A handle on ref r (counted for the live-gate filter of flush)."""
        self._dag.hinc(r >> 1)
        return _Bit(self, r, level, trivial)

    def encrypt(self, b):
        """Fresh encryption of bit b (all lanes) — SimContext.encrypt, backend.py:178-181."""
        if b not in (0, 1):
            raise ValueError(f"plaintext bit must be 0 or 1, got {b!r}")
        return self.encrypt_lanes(np.full(self.lanes, int(b), np.uint8))

    def encrypt_lanes(self, bits):
        """Fresh encryption of one bit per lane (len(bits) == lanes)."""
        bits = np.asarray(bits)
        if bits.shape != (self.lanes,):
            raise ValueError(f"expected {self.lanes} lane bits, got shape {bits.shape}")
        if not np.all((bits == 0) | (bits == 1)):
            raise ValueError("plaintext bits must be 0 or 1")
        with self._lock:
            idx0 = self._enc_count
            self._enc_count += self.lanes
            cts = self._encrypt_host(bits.astype(np.uint8), idx0)
            nid = self._dag.add_input()  # value known on the host; uploaded at flush
            self._inputs[nid] = cts
            return self._bit(nid << 1, 0)

    def encrypt_many(self, bits):
        """Vectorised encrypt: bits shape [count] (broadcast over lanes) or
        [count, lanes]; returns a list of handles."""
        bits = np.asarray(bits)
        if bits.ndim == 1:
            bits = np.repeat(bits[:, None], self.lanes, axis=1)
        if bits.ndim != 2 or bits.shape[1] != self.lanes:
            raise ValueError(f"expected [count, {self.lanes}] bits")
        if not np.all((bits == 0) | (bits == 1)):
            raise ValueError("plaintext bits must be 0 or 1")
        count = bits.shape[0]
        with self._lock:
            idx0 = self._enc_count
            self._enc_count += count * self.lanes
            cts = self._encrypt_host(bits.reshape(-1).astype(np.uint8), idx0).reshape(count, self.lanes, -1)
            out = []
            for i in range(count):
                nid = self._dag.add_input()
                self._inputs[nid] = cts[i]
                out.append(self._bit(nid << 1, 0))
            return out

    def import_ciphertexts(self, cts):
        """Wrap existing LWE samples (e.g. all-gathered from other ranks) as
        level-0 handles: cts [count][lanes][n+1] (or [count][n+1] for lanes == 1)."""
        cts = np.asarray(cts, dtype=np.uint32)
        if cts.ndim == 2:
            cts = cts[:, None, :]
        if cts.shape[1:] != (self.lanes, self.params.n + 1):
            raise ValueError(f"expected [count, {self.lanes}, {self.params.n + 1}] ciphertexts, got {cts.shape}")
        with self._lock:
            out = []
            for i in range(cts.shape[0]):
                nid = self._dag.add_input()
                self._inputs[nid] = np.ascontiguousarray(cts[i])
                out.append(self._bit(nid << 1, 0))
            return out

    def export_ciphertexts(self, handles):
        """LWE samples of handles -> [count][lanes][n+1] (NOT flags applied;
        constants become noiseless trivial samples)."""
        self._check(*handles)
        with self._lock:
            refs = [h._value for h in handles]
            for r in refs:
                self._dag.revive(r >> 1)
            if self._dag.pending_count():
                self.flush()
            out = np.zeros((len(refs), self.lanes, self.params.n + 1), np.uint32)
            live = [i for i, r in enumerate(refs) if (r >> 1) != 0]
            if live:
                out[live] = self._ciphertexts([refs[i] for i in live])
            for i, r in enumerate(refs):
                if (r >> 1) == 0:
                    out[i, :, -1] = EIGHTH if r & 1 else (-EIGHTH) & MASK32
                elif r & 1:
                    out[i] = (0 - out[i].astype(np.int64)).astype(np.uint32)
            return out

    def export_ciphertexts_device(self, handles):
        """export_ciphertexts into a torch.int32 CUDA tensor [count][lanes][n+1]
        on this context's GPU, without host staging (multi-GPU exchange)."""
        import torch

        self._check(*handles)
        with self._lock:
            refs = [h._value for h in handles]
            for r in refs:
                self._dag.revive(r >> 1)
            if self._dag.pending_count():
                self.flush()
            self._join_bg()
            words = self.params.n + 1
            out = torch.zeros((len(refs), self.lanes, words), dtype=torch.int32, device=f"cuda:{self.device}")
            host_inputs = [i for i, r in enumerate(refs) if (r >> 1) in self._inputs]
            dev = [i for i, r in enumerate(refs) if (r >> 1) != 0 and (r >> 1) not in self._inputs]
            if dev:
                eng = self._ensure_engine()
                slots = self._map_slots([(refs[i] >> 1) - 1 for i in dev])
                phys = (slots[:, None] * self.lanes + np.arange(self.lanes)[None, :]).reshape(-1)
                buf = torch.empty((len(dev) * self.lanes, words), dtype=torch.int32, device=out.device)
                eng.gather_device(phys.astype(np.uint32), buf.data_ptr(), words)
                out[dev] = buf.view(len(dev), self.lanes, words)
            for i in host_inputs:
                out[i] = torch.from_numpy(self._inputs[refs[i] >> 1].view(np.int32)).to(out.device)
            for i, r in enumerate(refs):
                if (r >> 1) == 0:
                    out[i, :, -1] = EIGHTH if r & 1 else -EIGHTH
                elif r & 1:
                    out[i] = -out[i]  # two's complement negation = mod-2^32 negation
            return out

    def import_ciphertexts_device(self, cts):
        """import_ciphertexts from a torch.int32 CUDA tensor [count][lanes][n+1]
        on this context's GPU: copied device-to-device into fresh pool slots."""
        with self._lock:
            if cts.dim() == 2:
                cts = cts[:, None, :]
            if tuple(cts.shape[1:]) != (self.lanes, self.params.n + 1):
                raise ValueError(f"expected [count, {self.lanes}, {self.params.n + 1}] ciphertexts, got {tuple(cts.shape)}")
            cts = cts.contiguous()
            nids = [self._dag.add_input() for _ in range(cts.shape[0])]
            if nids:
                eng = self._ensure_engine()
                # the engine copies on its own (non-blocking) stream: the producer of `cts`
                # (an NCCL all-gather, torch.cat, .contiguous()) ran on torch's current stream
                import torch

                torch.cuda.current_stream(cts.device).synchronize()
                phys = np.asarray(self._map_slots(np.asarray(nids, dtype=np.int64) - 1), dtype=np.int64)
                breaks = np.flatnonzero(np.diff(phys) != 1) + 1
                words = self.params.n + 1
                row = self.lanes * words * 4
                for run in np.split(np.arange(phys.size), breaks):
                    eng.put_device(int(phys[run[0]]) * self.lanes, run.size * self.lanes,
                                   cts.data_ptr() + int(run[0]) * row, words)
            return [self._bit(nid << 1, 0) for nid in nids]

    def _encrypt_host(self, bits, idx0):
        # one ChaCha stream per context; the ciphertext index continues across calls
        return self.keys.encrypt(bits, seed=self.enc_seed, stream=self.enc_stream, first_index=idx0)

    def trivial_const(self, b):
        """SimContext.trivial_const (backend.py:183-186): public, free, level 0."""
        if b not in (0, 1):
            raise ValueError(f"plaintext bit must be 0 or 1, got {b!r}")
        return self._bit(int(b), 0, int(b))

    # -- gates -------------------------------------------------------------------

    def _binary_gate(self, kind, a, b):
        """SimContext._binary_gate (backend.py:205-209) on real ciphertexts."""
        if not (isinstance(a, CipherBit) and isinstance(b, CipherBit) and a._ctx is self and b._ctx is self):
            raise ContextMismatchError("bit handle does not belong to this context")
        la, lb = a.level, b.level
        level = (la if la > lb else lb) + 1
        with self._lock:
            self.global_stats.record(kind, level)
            for scope in self._scopes:
                scope.record(kind, level)
            r = self._dag.gate(_KIND[kind], a._value, b._value)  # counts the handle below
            if self.stream_at:
                self._tick -= 1
                if self._tick <= 0:
                    if kind is XOR or kind is XNOR:
                        # a half adder issues its AND right after its XOR (circuits.py:95-98):
                        # check again after the next gate, so that a background flush never
                        # starts between the two and the pair stays one HA record
                        self._tick = 1
                    else:
                        self._tick = self._tick_every
                        self._maybe_stream()
            return _Bit(self, r, level)

    def g_and(self, a, b):
        return self._binary_gate(AND, a, b)

    def g_or(self, a, b):
        return self._binary_gate(OR, a, b)

    def g_xor(self, a, b):
        return self._binary_gate(XOR, a, b)

    def g_xnor(self, a, b):
        return self._binary_gate(XNOR, a, b)

    def g_not(self, a):
        """SimContext.g_not (backend.py:223-228): free sign flip."""
        self._check(a)
        if not _ref_backend.NOT_IS_FREE:
            return self.g_xnor(a, self.trivial_const(0))
        trivial = None if a.trivial_value is None else 1 - a.trivial_value
        with self._lock:
            return self._bit(a._value ^ 1, a.level, trivial)

    def g_mux(self, s, a, b):
        """SimContext.g_mux (backend.py:230-237)."""
        self._check(s, a, b)
        if s.trivial_value is not None:
            return a if s.trivial_value else b
        level = max(s.level, a.level, b.level) + 1
        with self._lock:
            self._record(MUX, level)
            r = self._dag.mux(s._value, a._value, b._value)  # counts the handle below
            if self.stream_at:
                self._tick -= 1
                if self._tick <= 0:
                    self._tick = self._tick_every
                    self._maybe_stream()
            return _Bit(self, r, level)

    # -- carry-save popcount (opt-in, popcount.py) ------------------------------

    def _csa_popcount(self, bits, out_levels):
        """Handles (LSB first, levels `out_levels`) on the binary digits of the
        number of true bits, built natively as a compressor network (Dag.csa);
        None if the network does not have exactly len(out_levels) non-constant
        digits (duplicate operands), in which case nothing live was created."""
        refs = np.fromiter((b._value for b in bits), dtype=np.int64, count=len(bits))
        with self._lock:
            out = [int(r) for r in self._dag.csa(refs, self.csa_block)]
            handles = [_Bit(self, r, 0) for r in out]  # own the counted handles (dropped on return None)
            if len(out) != len(out_levels) or any((r >> 1) == 0 for r in out):
                return None
            for h, lvl in zip(handles, out_levels):
                h.level = lvl
            if self.stream_at:
                self._tick -= 2 * len(bits)
                if self._tick <= 0:
                    self._tick = self._tick_every
                    self._maybe_stream()
            return handles

    def _merge_stats(self, delta):
        """Add a GateStats' counts and level histogram to the global stats and every open scope."""
        with self._lock:
            for st in (self.global_stats, *self._scopes):
                for k, v in delta.counts.items():
                    st.counts[k] += v
                hist = st.level_histogram
                for lvl, c in delta.level_histogram.items():
                    hist[lvl] = hist.get(lvl, 0) + c

    # -- scoped stats (backend.py:241-257) --------------------------------------

    def begin_scope(self, label=""):
        with self._lock:
            self._scopes.append(GateStats(label=label))

    def end_scope(self):
        with self._lock:
            if not self._scopes:
                raise ScopeError("end_scope without matching begin_scope")
            return self._scopes.pop()

    @property
    def scope_depth(self):
        return len(self._scopes)

    @property
    def gate_count(self):
        return self.global_stats.total

    # -- execution ------------------------------------------------------------------

    def pending_count(self):
        return self._dag.pending_count()

    def schedule(self):
        """(level, records) batches the next flush would launch."""
        with self._lock:
            return self._build_schedule(self._dag.live(False))

    def _build_schedule(self, pending):
        """Level batches of hb_gate records for node ids `pending` (int64 array)."""
        ids = np.asarray(pending, dtype=np.int64)
        if ids.size == 0:
            return []
        op, a, b, c, lvl = self._dag.gather(ids)
        dst, s_a, s_b, s_c = ids - 1, (a >> 1) - 1, (b >> 1) - 1, (c >> 1) - 1
        is_and = op == _OP_AND
        is_xor = op == _OP_XOR
        is_mux = op == _OP_MUX
        is_maj = op == _OP_MAJ
        is_x3 = op == _OP_XOR3
        three = is_mux | is_maj | is_x3
        recs = np.zeros(op.size, dtype=GATE_DTYPE)
        recs["dst"] = self._map_slots(dst)
        recs["src_a"] = self._map_slots(s_a)
        recs["src_b"] = self._map_slots(s_b)
        # MUX records: src_a = selector, src_b = a, src_c = b (refs a/b/c of the node)
        recs["src_c"] = np.where(three, self._map_slots(np.where(s_c >= 0, s_c, 0)), 0)
        sa = 1 - 2 * (a & 1)
        sb = 1 - 2 * (b & 1)
        sc = 1 - 2 * (c & 1)
        recs["kind"] = np.where(is_mux, GATE_MUX, np.where(is_maj | is_x3, GATE_LIN3, GATE_LIN2))
        recs["c0"] = np.where(is_and, _C_AND, np.where(is_xor, _C_XOR, 0)).astype(np.uint32)
        # AND: signs of the refs; XOR: 2, 2; MUX: selector positive, alpha/beta = signs of a / b;
        # MAJ: signs of the three refs (c0 0); XOR3: -2, -2, -2 (c0 0: the doubled sum is
        # +-1/4 with the sign carrying the parity)
        recs["alpha"] = np.where(is_and | is_maj, sa, np.where(is_xor, 2, np.where(is_x3, -2, sb)))
        recs["beta"] = np.where(is_and | is_maj, sb, np.where(is_xor, 2, np.where(is_x3, -2, sc)))
        recs["gamma"] = np.where(is_maj, sc, np.where(is_x3, -2, 0))
        if self.fuse_half_adders:
            keep = self._fuse_half_adders(recs, is_and, is_xor, a >> 1, b >> 1)
            if keep is not None:
                recs, lvl = recs[keep], lvl[keep]
        order = np.argsort(lvl, kind="stable")
        lvl_sorted = lvl[order]
        bounds = np.flatnonzero(np.diff(lvl_sorted)) + 1
        out = []
        for chunk in np.split(order, bounds):
            out.append((int(lvl[chunk[0]]), recs[chunk]))
        return out

    @staticmethod
    def _fuse_half_adders(recs, is_and, is_xor, na, nb):
        """Pair every XOR node with an AND node (AND/OR of literals) on the same
        two operand nodes, rewrite the AND record into an HA record
        whose second output (src_c) is the XOR node's slot, and return the mask
        of records to keep (None: no pair).  XOR(la, lb) = XOR(a, b) xor
        [alpha < 0] xor [beta < 0], so gamma = alpha * beta makes the second
        output the XOR node's own value."""
        ia, ix = np.flatnonzero(is_and), np.flatnonzero(is_xor)
        if ia.size == 0 or ix.size == 0:
            return None
        # both nodes of a pair have level 1 + max(operand levels): the operand pair is the key
        lo, hi = np.minimum(na, nb).astype(np.int64), np.maximum(na, nb).astype(np.int64)
        key = lo * (int(hi.max()) + 1) + hi
        ka, first = np.unique(key[ia], return_index=True)  # one AND per operand pair
        _, pos_x, pos_a = np.intersect1d(key[ix], ka, assume_unique=False, return_indices=True)
        if pos_x.size == 0:
            return None
        xi, ai = ix[pos_x], ia[first[pos_a]]
        recs["kind"][ai] = GATE_HA
        recs["src_c"][ai] = recs["dst"][xi]
        recs["gamma"][ai] = recs["alpha"][ai] * recs["beta"][ai]
        keep = np.ones(recs.size, dtype=bool)
        keep[xi] = False
        return keep

    def flush(self):
        """Execute every pending gate on the device (level by level)."""
        with self._lock:
            self._launch(wait=True)

    def _maybe_stream(self):
        """Streaming flush: once `stream_at` gates are pending and the previous
        background batch is done, run them on a background thread while the
        caller keeps building the DAG (device work overlaps host Python)."""
        if (self.stream_at and self._dag.pending_count() >= self.stream_at
                and (self._bg is None or not self._bg.is_alive())):
            self._launch(wait=False)

    def _join_bg(self):
        bg, self._bg = self._bg, None
        if bg is not None:
            bg.join()
            if self._bg_error:
                exc = self._bg_error.pop()
                self._bg_error.clear()
                raise DeviceError(str(exc)) from exc

    @staticmethod
    def _run_batches(eng, batches, lanes, errors):
        try:
            for _lvl, recs in batches:
                eng.run_gates(recs, lanes=lanes)
            eng.sync()
        except RuntimeError as exc:
            errors.append(exc)

    def _launch(self, wait):
        # a background batch is only started when the previous one has finished; a
        # final (waiting) flush prepares its schedule while that batch still runs
        # and joins it just before launching (stream order does the rest)
        if not wait:
            self._join_bg()
        t0 = time.perf_counter()
        eng = self._ensure_engine()
        if self._inputs:
            self._upload_inputs(eng, list(self._inputs), [self._inputs[nid] for nid in self._inputs])
            self._inputs.clear()
        pending = self._dag.live(True)  # the rest of the pending gates become dormant
        if not wait and self.stream_min_width:
            pending, deferred = self._select_wide(pending)
            self._dag.requeue(deferred)
        if pending.size == 0:
            if wait:
                self._join_bg()
            return
        batches = self._build_schedule(pending)
        self._history.extend(batches)
        self._dag.mark_done(pending)  # results are read only after _join_bg
        n_mux = sum(int(np.count_nonzero(r["kind"] == GATE_MUX)) for _, r in batches)
        n_ha = sum(int(np.count_nonzero(r["kind"] == GATE_HA)) for _, r in batches)
        self.exec_stats["gates"] += int(pending.size) * self.lanes
        self.exec_stats["bootstraps"] += (int(pending.size) + n_mux - n_ha) * self.lanes
        self.exec_stats["half_adders"] = self.exec_stats.get("half_adders", 0) + n_ha * self.lanes
        self.exec_stats["levels"] += len(batches)
        self.exec_stats["flushes"] += 1
        if wait:
            self._join_bg()
            errors = []
            self._run_batches(eng, batches, self.lanes, errors)
            if errors:
                raise DeviceError(str(errors[0])) from errors[0]
        else:
            self._bg = threading.Thread(target=self._run_batches, args=(eng, batches, self.lanes, self._bg_error),
                                        daemon=True)
            self._bg.start()
        self.exec_stats["flush_s"] += time.perf_counter() - t0

    def _select_wide(self, pending):
        """Split a background flush's live pending gates into (run, deferred):
        level by level, the gates whose operands are all done or run in this
        flush run if there are at least `stream_min_width` bootstraps of them;
        otherwise they, and everything depending on them, are deferred."""
        if pending.size == 0:
            return pending, pending
        op, a, b, c, lvl = self._dag.gather(pending)
        blocked = np.zeros(self._dag.size(), dtype=bool)
        run = np.zeros(pending.size, dtype=bool)
        order = np.argsort(lvl, kind="stable")
        bounds = np.flatnonzero(np.diff(lvl[order])) + 1
        cost = 1 + (op == _OP_MUX)  # bootstraps per record
        for idx in np.split(order, bounds):
            ok = ~(blocked[a[idx] >> 1] | blocked[b[idx] >> 1] | blocked[c[idx] >> 1])
            if int(cost[idx][ok].sum()) * self.lanes >= self.stream_min_width:
                run[idx[ok]] = True
                blocked[pending[idx[~ok]]] = True
            else:
                blocked[pending[idx]] = True
        return pending[run], pending[~run]

    def _upload_inputs(self, eng, nids, cts):
        """Host ciphertexts of input nodes -> their pool slots, one copy per run
        of consecutive physical slots (inputs are allocated in order)."""
        phys = np.asarray(self._map_slots(np.asarray(nids, dtype=np.int64) - 1), dtype=np.int64)
        order = np.argsort(phys, kind="stable")
        phys = phys[order]
        breaks = np.flatnonzero(np.diff(phys) != 1) + 1
        for run in np.split(np.arange(phys.size), breaks):
            block = np.stack([np.asarray(cts[order[i]], np.uint32).reshape(self.lanes, -1) for i in run])
            eng.upload(int(phys[run[0]]) * self.lanes, block.reshape(run.size * self.lanes, -1))

    def replay(self, handles, cts):
        """Per-model DAG caching: the circuit is data-oblivious,
        so after one evaluation the recorded level schedule can be re-run on new
        encrypted inputs without rebuilding the Python DAG.  `handles` are input
        handles of this context (from encrypt*/import_ciphertexts), `cts` their
        new ciphertexts [count][lanes][n+1] (or [count][n+1] for lanes == 1).
        Every handle derived from them decrypts to the new results afterwards."""
        self._check(*handles)
        cts = np.asarray(cts, dtype=np.uint32)
        if cts.ndim == 2:
            cts = cts[:, None, :]
        if cts.shape != (len(handles), self.lanes, self.params.n + 1):
            raise ValueError(f"expected [{len(handles)}, {self.lanes}, {self.params.n + 1}] ciphertexts")
        with self._lock:
            if self._dag.pending_count():
                self.flush()
            nids = [h._value >> 1 for h in handles]
            if any(nid == 0 or self._dag.op(nid) != _OP_INPUT for nid in nids) or any(h._value & 1 for h in handles):
                raise ValueError("replay inputs must be (non-negated) input handles")
            self._join_bg()
            t0 = time.perf_counter()
            eng = self._ensure_engine()
            self._inputs.clear()
            self._upload_inputs(eng, nids, list(cts))
            try:
                for _lvl, recs in self._replay_schedule():
                    eng.run_gates(recs, lanes=self.lanes)
                eng.sync()
            except RuntimeError as exc:
                raise DeviceError(str(exc)) from exc
            self.exec_stats["replays"] = self.exec_stats.get("replays", 0) + 1
            self.exec_stats["flush_s"] += time.perf_counter() - t0

    def compile_schedule(self, inputs, outputs, meta=None):
        """Compile once, serve many: the level schedule this
        context executed, in logical slots, with the slot maps of `inputs`
        (non-negated input handles) and `outputs` (any handles).  A fresh
        context runs it on new ciphertexts with `run_schedule` without the
        reference compiler or the gate DAG.  The schedule is key-independent."""
        self._check(*inputs, *outputs)
        with self._lock:
            live = [h._value >> 1 for h in outputs if (h._value >> 1) != 0]
            for nid in live:
                self._dag.revive(nid)
            if self._dag.pending_count() or any(not self._dag.is_done(nid) for nid in live):
                self.flush()
            self._join_bg()
            nids = [h._value >> 1 for h in inputs]
            if any(nid == 0 or self._dag.op(nid) != _OP_INPUT for nid in nids) or any(h._value & 1 for h in inputs):
                raise ValueError("schedule inputs must be (non-negated) input handles")
            levels = []
            for _lvl, recs in self._replay_schedule():
                r = recs.copy()
                for f in Schedule.SLOT_FIELDS:
                    r[f] = self._unmap_slots(recs[f])
                levels.append(r)
            out_refs = np.array([h._value for h in outputs], dtype=np.int64)
            ins = np.array(nids, dtype=np.int64) - 1
            outs = (out_refs >> 1) - 1  # -1: a public constant
            used = [ins, outs] + [r[f].astype(np.int64) for r in levels for f in Schedule.SLOT_FIELDS]
            n_slots = int(max((int(u.max()) for u in used if u.size), default=-1)) + 1
            return Schedule(levels, ins, outs, (out_refs & 1).astype(np.uint8), n_slots, self.lanes,
                            self.params.n, dict(meta or {}, counted=self.global_stats.as_dict()))

    def run_schedule(self, sched, cts):
        """Run a compiled schedule on new input ciphertexts `cts` [inputs][lanes][n+1]
        (or [inputs][n+1] for lanes == 1); returns the output ciphertexts
        [outputs][lanes][n+1] (NOT flags applied, constants as trivial samples).
        Uses pool chunks of its own: the context's DAG is untouched."""
        if sched.lanes != self.lanes or sched.n != self.params.n:
            raise ValueError(f"schedule compiled for lanes={sched.lanes}, n={sched.n}; "
                             f"context has lanes={self.lanes}, n={self.params.n}")
        cts = np.asarray(cts, dtype=np.uint32)
        if cts.ndim == 2:
            cts = cts[:, None, :]
        if cts.shape != (sched.inputs.size, self.lanes, self.params.n + 1):
            raise ValueError(f"expected [{sched.inputs.size}, {self.lanes}, {self.params.n + 1}] ciphertexts")
        with self._lock:
            self._join_bg()
            t0 = time.perf_counter()
            eng = self._ensure_engine()
            mp = lambda v: self._map_slots(v, self._sched_chunks, sched.n_slots)  # noqa: E731
            phys = np.asarray(mp(sched.inputs), dtype=np.int64)
            order = np.argsort(phys, kind="stable")
            ps = phys[order]
            breaks = np.flatnonzero(np.diff(ps) != 1) + 1
            try:
                for run in np.split(np.arange(ps.size), breaks):
                    block = cts[order[run]].reshape(run.size * self.lanes, -1)
                    eng.upload(int(ps[run[0]]) * self.lanes, block)
                for recs in sched.levels:
                    r = recs.copy()
                    for f in Schedule.SLOT_FIELDS:
                        r[f] = mp(recs[f].astype(np.int64))
                    eng.run_gates(r, lanes=self.lanes)
                out = np.zeros((sched.outputs.size, self.lanes, self.params.n + 1), np.uint32)
                var = np.flatnonzero(sched.outputs >= 0)
                if var.size:
                    op = np.asarray(mp(sched.outputs[var]), dtype=np.int64)
                    idx = (op[:, None] * self.lanes + np.arange(self.lanes)[None, :]).reshape(-1)
                    out[var] = eng.gather(idx.astype(np.uint32)).reshape(var.size, self.lanes, -1)
            except RuntimeError as exc:
                raise DeviceError(str(exc)) from exc
            const = sched.outputs < 0
            # public constants: trivial samples (0, +-1/8); NOT flags: mod-2^32 negation
            out[const, :, -1] = np.where(sched.out_neg[const, None] == 1, EIGHTH, (-EIGHTH) & MASK32)
            neg = (sched.out_neg == 1) & ~const
            out[neg] = np.uint32(0) - out[neg]
            self.exec_stats["schedule_runs"] = self.exec_stats.get("schedule_runs", 0) + 1
            self.exec_stats["flush_s"] += time.perf_counter() - t0
            return out

    def _replay_schedule(self):
        """The executed history regrouped by node level: streaming flushes split
        a model's levels over several launches; a replay runs each level once."""
        if getattr(self, "_replay_cache", (None,))[0] != len(self._history):
            if len(self._history) > 1:
                lv = np.concatenate([np.full(r.size, l, np.int64) for l, r in self._history])
                recs = np.concatenate([r for _, r in self._history])
                order = np.argsort(lv, kind="stable")
                bounds = np.flatnonzero(np.diff(lv[order])) + 1
                sched = [(int(lv[c[0]]), recs[c]) for c in np.split(order, bounds)]
            else:
                sched = list(self._history)
            self._replay_cache = (len(self._history), sched)
        return self._replay_cache[1]

    def _ciphertexts(self, refs):
        """Host LWE samples [len(refs)][lanes][n+1] for node refs (no negation)."""
        nodes = [r >> 1 for r in refs]
        out = np.zeros((len(nodes), self.lanes, self.params.n + 1), np.uint32)
        need = []
        for i, nid in enumerate(nodes):
            cts = self._inputs.get(nid)
            if cts is not None:
                out[i] = cts
            else:
                need.append(i)
        if need:
            self._join_bg()
            eng = self._ensure_engine()
            slots = self._map_slots([nodes[i] - 1 for i in need])
            phys = (slots[:, None] * self.lanes + np.arange(self.lanes)[None, :]).reshape(-1)
            try:
                got = eng.gather(phys.astype(np.uint32))
            except RuntimeError as exc:
                raise DeviceError(str(exc)) from exc
            out[need] = got.reshape(len(need), self.lanes, -1)
        return out

    def decrypt_lanes(self, c):
        """Decrypt one handle in every lane -> uint8 array [lanes]."""
        return self.decrypt_many([c])[0]

    def decrypt_many(self, handles):
        """Decrypt several handles with one device gather -> uint8 [count][lanes]."""
        self._check(*handles)
        with self._lock:
            refs = [h._value for h in handles]
            res = np.zeros((len(refs), self.lanes), np.uint8)
            live = [i for i, r in enumerate(refs) if (r >> 1) != 0]
            for i, r in enumerate(refs):
                if (r >> 1) == 0:
                    res[i] = r & 1
            if live:
                for i in live:
                    self._dag.revive(refs[i] >> 1)
                if self._dag.pending_count() or any(not self._dag.is_done(refs[i] >> 1) for i in live):
                    self.flush()
                cts = self._ciphertexts([refs[i] for i in live])
                bits = self.keys.decrypt(cts.reshape(-1, cts.shape[-1])).reshape(len(live), self.lanes)
                for j, i in enumerate(live):
                    res[i] = bits[j] ^ (refs[i] & 1)
            return res

    def decrypt(self, c):
        """SimContext.decrypt (backend.py:188-190): the flush point.  Returns an
        int for lanes == 1, else a uint8 array over lanes."""
        self._check(c)
        out = self.decrypt_many([c])[0]
        return int(out[0]) if self.lanes == 1 else out

    def phase(self, c):
        """Signed torus phase (int32 units of 2^-32) of a handle, per lane."""
        self._check(c)
        with self._lock:
            if (c._value >> 1) == 0:
                return None
            self._dag.revive(c._value >> 1)
            if self._dag.pending_count():
                self.flush()
            cts = self._ciphertexts([c._value])[0]
            ph = self.keys.phase(cts).astype(np.int64)
            return -ph if c._value & 1 else ph


class Schedule:
    """A compiled model (TfheContext.compile_schedule): executed level records
    in logical slots, input/output slot maps, lanes and n; save/load as .npz."""

    SLOT_FIELDS = ("dst", "src_a", "src_b", "src_c")

    def __init__(self, levels, inputs, outputs, out_neg, n_slots, lanes, n, meta):
        self.levels = list(levels)
        self.inputs = np.asarray(inputs, dtype=np.int64)
        self.outputs = np.asarray(outputs, dtype=np.int64)
        self.out_neg = np.asarray(out_neg, dtype=np.uint8)
        self.n_slots, self.lanes, self.n = int(n_slots), int(lanes), int(n)
        self.meta = meta

    @property
    def records(self):
        return sum(r.size for r in self.levels)

    def save(self, path):
        import json

        sizes = np.array([r.size for r in self.levels], dtype=np.int64)
        recs = np.concatenate(self.levels) if self.levels else np.zeros(0, GATE_DTYPE)
        hdr = json.dumps({"format": "hebnn-b200/schedule", "version": 1, "n_slots": self.n_slots,
                          "lanes": self.lanes, "n": self.n, "meta": self.meta})
        np.savez(path, header=np.frombuffer(hdr.encode(), np.uint8), records=recs, sizes=sizes,
                 inputs=self.inputs, outputs=self.outputs, out_neg=self.out_neg)

    @classmethod
    def load(cls, path):
        import json

        with np.load(path, allow_pickle=False) as z:
            hdr = json.loads(bytes(z["header"]).decode())
            if hdr.get("format") != "hebnn-b200/schedule" or hdr.get("version") != 1:
                raise ValueError("not a hebnn-b200 schedule document")
            recs = z["records"]
            if recs.dtype != GATE_DTYPE:
                raise ValueError("schedule records have the wrong layout")
            sizes = z["sizes"]
            if sizes.sum() != recs.size or (sizes < 0).any():
                raise ValueError("schedule level sizes do not match its records")
            n_slots = int(hdr["n_slots"])
            for f in cls.SLOT_FIELDS:
                if recs.size and int(recs[f].max()) >= n_slots:
                    raise ValueError("schedule record slot beyond n_slots")
            ins, outs = z["inputs"], z["outputs"]
            if (ins.size and (ins.min() < 0 or ins.max() >= n_slots)) or (outs.size and outs.max() >= n_slots):
                raise ValueError("schedule slot map beyond n_slots")
            levels = np.split(recs, np.cumsum(sizes)[:-1]) if sizes.size else []
            return cls(levels, ins, outs, z["out_neg"], n_slots, hdr["lanes"], hdr["n"], hdr["meta"])


__all__ = ["TfheContext", "DeviceError", "Schedule", "shared_keys", "shared_engine"]
