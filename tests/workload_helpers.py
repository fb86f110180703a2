"""Small helpers shared by multi-process test scripts."""
import numpy as np


def enc(tokens) -> bytes:
    """codec.hpp:15-22 encoding of a token list."""
    t = np.asarray(tokens, dtype=np.int64).astype("<u8")
    return np.uint64(len(t)).astype("<u8").tobytes() + t.tobytes()
