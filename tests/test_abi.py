"""CPU checks of the C-ABI library: it loads, exports every symbol the header
declares, refuses compute without a GPU (no CPU fallback), and its host-only
helpers (seeded init, codec, experience-store control plane) behave like the
reference."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2602_09578_b200 import _lib
from paper_2602_09578_b200.engine import seeded_weights, agent_seed

ROOT = Path(__file__).resolve().parent.parent


def declared_symbols():
    text = (ROOT / "include" / "flexmarl" / "cabi.h").read_text()
    return set(re.findall(r"^(?:const char\*|int|int64_t|uint64_t|void)\s+\*?(fm_\w+)\(", text, flags=re.M))


def test_header_symbols_exported():
    L = _lib.lib()
    decl = declared_symbols()
    assert len(decl) >= 50
    for s in decl:
        assert hasattr(L, s), s
    assert decl == set(_lib.EXPORTED)


def test_abi_version_and_status_names():
    L = _lib.lib()
    assert L.fm_abi_version() == 1
    assert L.fm_status_name(23).decode() == "VersionMismatch"
    assert L.fm_status_name(25).decode() == "IncompleteBatch"


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = C.c_void_p()
    st = _lib.lib().fm_ctx_create(0, C.byref(h))
    assert st == _lib.FM_ERR_NO_DEVICE


def test_seeded_weights_host_bit_exact():
    f = np.load(ROOT / "tests" / "golden" / "rng.npz")
    for a in ("planner", "executor"):
        assert np.array_equal(seeded_weights(32, 16, agent_seed(2048, a)), f[f"W0_{a}"])


def test_encode_tokens_matches_codec():
    from paper_2602_09578_b200 import workload as wl
    toks = np.array([0, 1, 31999, -1, 2 ** 31 - 1], np.int32)
    out = np.zeros(8 + 8 * len(toks), np.uint8)
    n = _lib.lib().fm_encode_tokens(toks.ctypes.data, len(toks), out.ctypes.data)
    assert n == len(out)
    assert out.tobytes() == wl.encode_tokens(toks)
    assert np.array_equal(wl.decode_tokens(out.tobytes()), toks)
