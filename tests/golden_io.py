"""Helpers to read the bit-exact JSON fixtures in tests/golden/."""
import json
import os
import struct

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def unhex(bits):
    """List of 16-hex-digit big-endian IEEE-754 patterns -> float64 array."""
    if not bits:
        return np.empty(0, dtype=np.float64)
    raw = b"".join(bytes.fromhex(b) for b in bits)
    return np.frombuffer(raw, dtype=">f8").astype(np.float64)


def same_bits(a, b) -> bool:
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and a.view(np.uint64).tobytes() == b.view(np.uint64).tobytes()


def sha256(a) -> str:
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()
