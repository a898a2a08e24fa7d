"""Exception classes mirroring the reference's (proj/include/mtc/errors.hpp:26-55)."""
from __future__ import annotations


class MtcError(RuntimeError):
    pass


class ParseError(MtcError):
    """Malformed circuit / plan / samples text (CLI exit 2)."""

    def __init__(self, what: str, line: int = 0):
        super().__init__(f"line {line}: {what}" if line else what)
        self.line = line


class DataError(MtcError):
    """Inconsistent inputs (CLI exit 2)."""


class MemoryCapError(MtcError):
    """The evaluation would exceed its memory cap (CLI exit 3)."""

    def __init__(self, what: str, node: int = -1):
        super().__init__(what)
        self.node = node


class EngineError(MtcError):
    """CUDA / internal failure inside the engine (CLI exit 1)."""
