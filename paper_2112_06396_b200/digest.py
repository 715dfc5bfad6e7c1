"""Canonical digests of residue arrays (golden fixtures, parity at scale)."""

from __future__ import annotations

import hashlib

import numpy as np


def digest(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        a = np.ascontiguousarray(np.asarray(a), dtype="<u8")
        h.update(str(a.shape).encode())
        h.update(a.tobytes())
    return h.hexdigest()
