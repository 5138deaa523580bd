"""Small helpers shared by the tests (no method arithmetic)."""
import os

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def read_golden(name):
    """Parse a tests/golden fixture: '#' comments, then 'key v1 v2 ...' lines."""
    out = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            key, *vals = line.split()
            out[key] = vals
    return out


def bits_from_dense(v):
    """Dense 0/1 vector -> little-endian uint32 bitmap words (ceil(n/32)), as int32 numpy."""
    import numpy as np
    v = np.asarray(v, dtype=np.uint8)
    n = len(v)
    nw = (n + 31) // 32
    pad = np.zeros(nw * 32, dtype=np.uint8)
    pad[:n] = v != 0
    return np.packbits(pad, bitorder="little").view("<u4").astype(np.uint32).view(np.int32)


def dense_from_bits(words, n):
    import numpy as np
    w = np.asarray(words).astype(np.int32).view(np.uint32).astype("<u4")
    return np.unpackbits(w.view(np.uint8), bitorder="little")[:n].astype(np.uint8)
