"""The reference's plugin interface for this path, re-exported.

`TfheContext` must be a drop-in for `hebnn.backend.SimContext`, so it uses the
reference's own `GateBackend` ABC, `CipherBit` handle, `GateStats`, error
types and gate-kind names (/root/reference/pkg/src/hebnn/backend.py:23-150)
whenever `hebnn` is importable (it is installed into baseline/_ref).  Without
it, identical mirrors are defined here (same names, fields and error
hierarchy), so the engine still works stand-alone.
"""

from __future__ import annotations

try:  # the reference package (baseline/_ref) — the real drop-in target
    from hebnn import backend as _ref_backend
    from hebnn.backend import (  # noqa: F401
        AND,
        COSTED_KINDS,
        MUX,
        OR,
        XNOR,
        XOR,
        CipherBit,
        ContextMismatchError,
        GateBackend,
        GateStats,
        ScopeError,
    )

    HAVE_REFERENCE = True

    def not_is_free():
        return _ref_backend.NOT_IS_FREE

except ImportError:  # pragma: no cover - exercised only without baseline/_ref
    import abc
    from dataclasses import dataclass, field

    HAVE_REFERENCE = False
    AND, OR, XOR, XNOR, MUX = "AND", "OR", "XOR", "XNOR", "MUX"
    COSTED_KINDS = (AND, OR, XOR, XNOR, MUX)
    NOT_IS_FREE = True

    def not_is_free():
        return NOT_IS_FREE

    class ContextMismatchError(ValueError):
        """A bit handle was used with a context that did not create it."""

    class ScopeError(RuntimeError):
        """begin_scope/end_scope calls were not properly balanced."""

    class CipherBit:
        __slots__ = ("_ctx", "_value", "level", "trivial_value")

        def __init__(self, ctx, value, level, trivial_value=None):
            self._ctx = ctx
            self._value = value
            self.level = level
            self.trivial_value = trivial_value

        @property
        def context(self):
            return self._ctx

        def __repr__(self):
            kind = "trivial" if self.trivial_value is not None else "cipher"
            return f"<CipherBit {kind} level={self.level}>"

    @dataclass
    class GateStats:
        label: str = ""
        counts: dict = field(default_factory=lambda: {k: 0 for k in COSTED_KINDS})
        level_histogram: dict = field(default_factory=dict)

        def record(self, kind, level):
            self.counts[kind] += 1
            self.level_histogram[level] = self.level_histogram.get(level, 0) + 1

        @property
        def total(self):
            return sum(self.counts.values())

        @property
        def max_level(self):
            return max(self.level_histogram) if self.level_histogram else 0

    class GateBackend(abc.ABC):
        @abc.abstractmethod
        def encrypt(self, b): ...

        @abc.abstractmethod
        def decrypt(self, c): ...

        @abc.abstractmethod
        def trivial_const(self, b): ...

        @abc.abstractmethod
        def g_and(self, a, b): ...

        @abc.abstractmethod
        def g_or(self, a, b): ...

        @abc.abstractmethod
        def g_xor(self, a, b): ...

        @abc.abstractmethod
        def g_xnor(self, a, b): ...

        @abc.abstractmethod
        def g_not(self, a): ...

        @abc.abstractmethod
        def g_mux(self, s, a, b): ...

        @abc.abstractmethod
        def begin_scope(self, label): ...

        @abc.abstractmethod
        def end_scope(self): ...
