"""GPU tests of the §8f "next" rows built this round:
  f1  weight publish / rollout sync (training.hpp:459-467, rollout.hpp:510-541)
  f2  byte-compatible PolicyState wire format (training.hpp:107-164)
"""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2602_09578_b200 import _lib
from fixture_runner import run_fixture, payload

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
L = _lib.lib


def _agent(ctx, V, D, W0, name=b"n", precision=_lib.PRECISION_BF16_TC):
    h = C.c_void_p()
    _lib.check(L().fm_agent_create(ctx.handle, name, V, D, precision, C.byref(h)))
    _lib.check(L().fm_agent_set_weights(h, np.ascontiguousarray(W0).ctypes.data))
    return h


def _train_step(ctx, h, f, update=True, n_mb=4):
    G, mb = int(f["G"]), int(f["mb"])
    po = f["poll_order"]
    for b in range(n_mb):
        idx = po[b * mb:(b + 1) * mb]
        arr = (_lib.fm_sample * mb)(*[_lib.fm_sample(ctx.put(payload(f, int(f["prompt_off"][i]))),
                                                     ctx.put(payload(f, int(f["resp_off"][i]))),
                                                     float(f["adv"][i])) for i in idx])
        t = C.c_int64()
        _lib.check(L().fm_train_micro_batch(h, arr, mb, G, C.byref(t)))
    if update:
        _lib.check(L().fm_apply_update(h, G, 1e-6, 0.9, 0.999, 1e-8, None, None))


def _serialize(h, G=64) -> bytes:
    n = C.c_uint64()
    _lib.check(L().fm_agent_serialize(h, G, None, 0, C.byref(n)))
    buf = (C.c_uint8 * n.value)()
    _lib.check(L().fm_agent_serialize(h, G, buf, n.value, C.byref(n)))
    return bytes(buf)


def test_serialize_byte_identical_to_reference(ctx):
    f = np.load(GOLD / "mid_agent0.npz")
    V, D = int(f["V"]), int(f["D"])
    ctx.reset_arena()
    h = _agent(ctx, V, D, f["W0"])
    try:
        _train_step(ctx, h, f)  # one full update: nothing pending, step 1, version 1
        ours = _serialize(h)
        W = np.empty(V * D)
        m = np.empty(V * D, np.float32)
        v = np.empty(V * D, np.float32)
        step = C.c_int64()
        _lib.check(L().fm_agent_read_weights(h, W.ctypes.data))
        _lib.check(L().fm_agent_read_moments(h, m.ctypes.data, v.ctypes.data, C.byref(step)))
        ref = orc.ref_serialize_state(1, step.value, 0, W.reshape(V, D), m.astype(np.float64).reshape(V, D),
                                      v.astype(np.float64).reshape(V, D))
        assert ours == ref
    finally:
        L().fm_agent_destroy(h)


def test_state_roundtrip_with_pending_gradient(ctx):
    f = np.load(GOLD / "mid_agent0.npz")
    V, D = int(f["V"]), int(f["D"])
    ctx.reset_arena()
    a = _agent(ctx, V, D, f["W0"], b"a")
    b = _agent(ctx, V, D, np.zeros((V, D)), b"b")
    try:
        _train_step(ctx, a, f, update=True)
        _train_step(ctx, a, f, update=False, n_mb=2)  # mid-step: 32 samples pending
        blob = _serialize(a)
        _lib.check(L().fm_agent_deserialize(b, 64, blob, len(blob)))
        ca, cb = C.c_uint64(), C.c_uint64()
        _lib.check(L().fm_agent_state_checksum(a, C.byref(ca)))
        _lib.check(L().fm_agent_state_checksum(b, C.byref(cb)))
        assert ca.value == cb.value
        assert L().fm_agent_samples_accumulated(b) == 32
    finally:
        L().fm_agent_destroy(a)
        L().fm_agent_destroy(b)


def test_reference_reads_our_state_when_square(ctx):
    """With V == D the reference's own deserialize (training.hpp:135-164) reads
    our bytes back exactly (for V != D it transposes — the defect at :146)."""
    V = D = 64
    W0 = np.random.default_rng(1).normal(size=(V, D))
    h = _agent(ctx, V, D, W0)
    try:
        blob = _serialize(h)
        r = orc.ref_deserialize_state(blob, V * D)
        assert r["rows"] == V and r["cols"] == D and r["version"] == 0 and r["cache_n"] == 0
        assert np.array_equal(r["W"], W0.reshape(-1))
    finally:
        L().fm_agent_destroy(h)


@pytest.mark.parametrize("dtype", [0, 1, 2])
def test_publish_weights_contiguous_buffer(ctx, dtype):
    import torch
    f = np.load(GOLD / "mid_agent0.npz")
    V, D = int(f["V"]), int(f["D"])
    ctx.reset_arena()
    h = _agent(ctx, V, D, f["W0"])
    w = C.c_void_p()
    try:
        _train_step(ctx, h, f)
        _lib.check(L().fm_publish_weights(h, dtype, C.byref(w)))
        ver, nb = C.c_int64(), C.c_uint64()
        _lib.check(L().fm_weights_info(w, C.byref(ver), None, None, None, C.byref(nb), None))
        assert ver.value == 1
        host = np.zeros(nb.value, np.uint8)
        _lib.check(L().fm_weights_get(w, host.ctypes.data, -1))  # one Get, one contiguous copy
        W = np.empty(V * D)
        _lib.check(L().fm_agent_read_weights(h, W.ctypes.data))
        if dtype == 0:  # pack_weights payload bytes (object_store.hpp:258-273)
            assert host.tobytes() == W.tobytes()
        elif dtype == 1:
            assert np.array_equal(host.view(np.float32), W.astype(np.float32))
        else:
            want = torch.tensor(W.astype(np.float32)).to(torch.bfloat16).view(torch.int16).numpy()
            assert np.array_equal(host.view(np.int16), want)
        # republish into the same buffer after another step: new version, new bytes
        _train_step(ctx, h, f)
        _lib.check(L().fm_publish_into(h, w))
        _lib.check(L().fm_weights_info(w, C.byref(ver), None, None, None, None, None))
        assert ver.value == 2
        w2 = C.c_void_p()
        _lib.check(L().fm_publish_weights(h, dtype, C.byref(w2)))
        fresh = np.zeros(nb.value, np.uint8)
        _lib.check(L().fm_weights_get(w2, fresh.ctypes.data, -1))
        L().fm_weights_destroy(w2)
        _lib.check(L().fm_weights_get(w, host.ctypes.data, -1))
        assert host.tobytes() == fresh.tobytes()
    finally:
        if w:
            L().fm_weights_destroy(w)
        L().fm_agent_destroy(h)
