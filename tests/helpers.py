"""Shared test helpers (no oracle imports here; tests pass checkers in)."""
import hashlib

import numpy as np


def tri_row(L: int, s: int, t: int) -> int:
    return s * L - s * (s - 1) // 2 + (t - s)


def table_digest(o, k, v) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(o, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(k, dtype="i1").tobytes())
    h.update(np.ascontiguousarray(v, dtype="<i4").tobytes())
    return h.hexdigest()


def ops_digest(ops) -> str:
    return hashlib.sha256(np.array(ops, dtype="<i4").reshape(-1).tobytes()).hexdigest()
