from ._lib import ConfigError, SolveError  # noqa: F401

__all__ = ["api", "synth"]
