"""ctypes binding of the C-ABI library (include/hg_gnn.h -> libhg_gnn.so).

Signatures are derived from the public header itself, so the header is the
single source of truth; ``exported_symbols()``/``declared_symbols()`` back the
CPU test that the library exports everything the header declares.

There is no CPU fallback: if the library cannot be loaded the import of any
compute entry point raises ``BackendUnavailable`` — loudly.
"""

from __future__ import annotations

import ctypes
import re
import threading
from pathlib import Path

from . import build as _build

HEADER = _build.INCLUDE / "hg_gnn.h"

_CTYPES = {
    "int": ctypes.c_int,
    "int32_t": ctypes.c_int32,
    "int64_t": ctypes.c_int64,
    "uint32_t": ctypes.c_uint32,
    "uint64_t": ctypes.c_uint64,
    "float": ctypes.c_float,
    "double": ctypes.c_double,
    "void": None,
}


class BackendUnavailable(RuntimeError):
    """The sm_100a library (or a CUDA device) is missing; no fallback exists."""


class HgError(RuntimeError):
    def __init__(self, fn, rc, msg):
        super().__init__(f"{fn} failed ({rc}): {msg}")
        self.fn, self.rc, self.msg = fn, rc, msg


def parse_header(path: Path = HEADER) -> dict:
    """{name: (restype, [argtypes])} for every hg_* prototype in the header."""
    text = re.sub(r"/\*.*?\*/", " ", path.read_text(), flags=re.S)
    text = re.sub(r"//[^\n]*", " ", text)
    out = {}
    for m in re.finditer(r"\b(int|int32_t|int64_t|uint32_t|uint64_t|void)\s+(hg_\w+)\s*\(([^;]*?)\)\s*;", text,
                         flags=re.S):
        ret, name, args = m.group(1), m.group(2), m.group(3).strip()
        argtypes = []
        if args and args != "void":
            for a in args.split(","):
                a = " ".join(a.split())
                if "*" in a:
                    argtypes.append(ctypes.c_void_p)
                else:
                    base = a.replace("const ", "").split()[0]
                    argtypes.append(_CTYPES[base])
        out[name] = (_CTYPES[ret], argtypes)
    return out


def declared_symbols() -> list[str]:
    return sorted(parse_header())


_lock = threading.Lock()
_lib = None


def load(build_if_missing: bool = True):
    """Load libhg_gnn.so (building it in-tree first if needed)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = _build.LIB
        if not path.exists() or _build._stale():
            if not build_if_missing:
                raise BackendUnavailable(f"{path} not built")
            try:
                _build.build()
            except Exception as exc:  # pragma: no cover - depends on toolchain
                if not path.exists():
                    raise BackendUnavailable(f"cannot build {path}: {exc}") from exc
        lib = ctypes.CDLL(str(path))
        for name, (res, args) in parse_header().items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def exported_symbols() -> list[str]:
    lib = load()
    return [n for n in declared_symbols() if hasattr(lib, n)]


def last_error() -> str:
    lib = load()
    buf = ctypes.create_string_buffer(1024)
    lib.hg_last_error(buf, 1024)
    return buf.value.decode(errors="replace")


def call(name: str, *args):
    """Invoke an int-returning entry point and raise HgError on failure."""
    fn = getattr(load(), name)
    rc = fn(*args)
    if rc != 0:
        raise HgError(name, rc, last_error())
    return rc


def fn(name: str):
    return getattr(load(), name)
