"""Edge cases of the micro-batch path against the f64 restatement (oracle,
pinned to the reference): empty responses (no rows), empty prompts (a first
token with an empty context: phi = 0, uniform softmax, no gradient),
out-of-range action tokens (never match a vocab row: -c p without the delta
term, policy.hpp:84-85), negative tokens in the context (feature = token mod D
through size_t, policy.hpp:48), one-token and long responses, a zero
advantage, a micro-batch with no rows at all, ragged micro-batches.  Both
precisions; tolerances as tests/test_gpu_path.py."""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2602_09578_b200 import _lib
import workload_helpers as wh

pytestmark = pytest.mark.gpu
L = _lib.lib


def rel_fro(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def _samples(V, rng):
    i32 = lambda x: np.asarray(x, np.int32)  # noqa: E731
    return [
        (i32(rng.integers(0, V, 5)), i32([])),                                # empty response: no rows
        (i32([]), i32(rng.integers(0, V, 7))),                                # empty prompt: n = 0 at t = 0
        (i32(rng.integers(0, V, 3)), i32([V + 3, -2, 2**31 - 1, 5, V])),       # actions outside [0, V)
        (i32([-7, -1, 2**31 - 1]), i32(rng.integers(0, V, 9))),               # negative / huge context tokens
        (i32(rng.integers(0, V, 4)), i32(rng.integers(0, V, 1))),             # one-token response
        (i32(rng.integers(0, V, 6)), i32(rng.integers(0, V, 300))),           # long response
        (i32(rng.integers(0, V, 2)), i32(rng.integers(0, V, 11))),            # (zero advantage below)
        (i32(rng.integers(0, V, 8)), i32(rng.integers(0, V, 40))),
    ]


def _run(ctx, precision, V, D, samples, adv, mb_sizes, lr):
    G = len(samples)
    h = C.c_void_p()
    _lib.check(L().fm_agent_create(ctx.handle, b"edge", V, D, precision, C.byref(h)))
    W0 = np.ascontiguousarray(np.random.default_rng(5).normal(size=(V, D)) * 0.5)
    try:
        _lib.check(L().fm_agent_set_weights(h, W0.ctypes.data))
        i = 0
        for n in mb_sizes:
            arr = (_lib.fm_sample * max(n, 1))(*[_lib.fm_sample(ctx.put(wh.enc(p)), ctx.put(wh.enc(r)), float(a))
                                                 for (p, r), a in zip(samples[i:i + n], adv[i:i + n])])
            t = C.c_int64()
            _lib.check(L().fm_train_micro_batch(h, arr, n, G, C.byref(t)))
            i += n
        _lib.check(L().fm_agent_sync(h))
        g = np.empty(V * D)
        _lib.check(L().fm_agent_read_grad(h, g.ctypes.data))
        gn = C.c_double()
        _lib.check(L().fm_apply_update(h, G, lr, 0.9, 0.999, 1e-8, C.byref(gn), None))
        W = np.empty(V * D)
        _lib.check(L().fm_agent_read_weights(h, W.ctypes.data))
        return W0, g.reshape(V, D), W.reshape(V, D), gn.value
    finally:
        L().fm_agent_destroy(h)


@pytest.mark.parametrize("precision", [_lib.PRECISION_BF16_TC, _lib.PRECISION_PARITY_F64])
@pytest.mark.parametrize("mb_sizes", [(4, 4), (3, 5), (1, 7), (8,)])  # ragged micro-batches
def test_edge_samples_match_reference(ctx, precision, mb_sizes):
    ctx.reset_arena()
    V, D = 300, 72
    rng = np.random.default_rng(17)
    samples = _samples(V, rng)
    adv = rng.normal(size=len(samples))
    adv[6] = 0.0
    lr = 1e-3
    W0, g, W, gn = _run(ctx, precision, V, D, samples, adv, mb_sizes, lr)
    ref = orc.run_agent(V, D, len(samples), len(samples), 1, samples, adv, W0, lr=lr)
    g_ref, dW_ref = ref["last_grad"], ref["W"] - W0
    if precision == _lib.PRECISION_PARITY_F64:
        assert rel_fro(g, g_ref) <= 1e-9
        assert rel_fro(W - W0, dW_ref) <= 1e-6
        assert abs(gn - ref["upd_grad_norm"][0]) <= 1e-9 * ref["upd_grad_norm"][0]
    else:
        assert rel_fro(g, g_ref) <= 2e-2
        cos = float((g * g_ref).sum() / (np.linalg.norm(g) * np.linalg.norm(g_ref)))
        assert cos >= 0.999
        assert rel_fro(W - W0, dW_ref) <= 5e-2
        assert abs(gn - ref["upd_grad_norm"][0]) <= 2e-2 * ref["upd_grad_norm"][0]


@pytest.mark.parametrize("precision", [_lib.PRECISION_BF16_TC, _lib.PRECISION_PARITY_F64])
def test_micro_batch_without_rows(ctx, precision):
    """Every response empty: the micro-batch counts toward G but trains no rows."""
    ctx.reset_arena()
    V, D = 300, 72
    rng = np.random.default_rng(3)
    samples = [(rng.integers(0, V, 4).astype(np.int32), np.zeros(0, np.int32)) for _ in range(4)]
    samples += _samples(V, rng)[3:7]
    adv = rng.normal(size=len(samples))
    W0, g, W, gn = _run(ctx, precision, V, D, samples, adv, (4, 4), 1e-3)
    ref = orc.run_agent(V, D, len(samples), len(samples), 1, samples, adv, W0, lr=1e-3)
    assert rel_fro(g, ref["last_grad"]) <= (1e-9 if precision == _lib.PRECISION_PARITY_F64 else 2e-2)
