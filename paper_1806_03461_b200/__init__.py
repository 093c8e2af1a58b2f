"""B200-native TFHE/CGGI gate-bootstrapping engine behind the reference
hebnn ``GateBackend``."""

__version__ = "0.1.0"
