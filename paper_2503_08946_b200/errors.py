"""Error model mirroring the reference's ``raceset::Error{ErrorKind}``
(/root/reference/proj/include/raceset/error.hpp:10-56; names from
src/affine.cpp:9-33).  ``str(Error)`` reads like the reference's
``what()``: "<kind name>: <message>".
"""
from __future__ import annotations

import enum


class ErrorKind(enum.Enum):
    # (reference enumerator, what() prefix) -- only the kinds this path raises,
    # plus the host-API kinds a C-ABI needs.
    SyntaxError = "syntax error"
    UnsupportedConstruct = "unsupported construct"
    StepLimitExceeded = "step limit exceeded"
    OutOfBounds = "out of bounds"
    CsrInvalid = "invalid csr"
    Io = "io error"
    InvalidArgument = "invalid argument"
    Cuda = "cuda error"
    Nccl = "nccl error"

    @property
    def label(self) -> str:
        return self.value


class Error(RuntimeError):
    def __init__(self, kind: ErrorKind, message: str, line: int = 0, col: int = 0):
        self.kind = kind
        self.line = line
        self.col = col
        if line:
            text = f"{line}:{col}: {kind.label}: {message}"
        else:
            text = f"{kind.label}: {message}"
        super().__init__(text)
