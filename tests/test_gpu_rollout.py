"""§8f-3: on-GPU rollout generation vs the reference's PolicyModel::generate.

The C1 golden fixtures' responses were produced by the compiled reference
(tests/datasets.py: ref_generate with the rollout.hpp:640-644 token seeds);
the GPU generator must reproduce them token for token, with log-probs within
1e-12 (fp64; only the exp/log ulps and the denominator order differ)."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

from paper_2602_09578_b200 import _lib
from paper_2602_09578_b200 import workload as wl
from fixture_runner import payload

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"
L = _lib.lib


def _dec(b):
    return wl.decode_tokens(b)


@pytest.mark.parametrize("layout", [0, 3])  # published f64 [V][D] or the transposed rollout layout
@pytest.mark.parametrize("name", ["c1_planner", "c1_executor"])
def test_generate_matches_reference(ctx, name, layout):
    f = np.load(GOLD / f"{name}.npz")
    agent = str(f["agent"])
    V, D = int(f["V"]), int(f["D"])
    h = C.c_void_p()
    _lib.check(L().fm_agent_create(ctx.handle, agent.encode(), V, D, _lib.PRECISION_PARITY_F64, C.byref(h)))
    W0 = np.ascontiguousarray(f["W0"])  # named: a temporary could be freed before the C call reads it
    _lib.check(L().fm_agent_set_weights(h, W0.ctypes.data))
    w = C.c_void_p()
    _lib.check(L().fm_publish_weights(h, layout, C.byref(w)))
    Wpub = np.zeros((V, D))
    if layout == 3:
        Wt = np.zeros((D, V))
        _lib.check(L().fm_weights_get(w, Wt.ctypes.data, -1))
        Wpub = np.ascontiguousarray(Wt.T)
    else:
        _lib.check(L().fm_weights_get(w, Wpub.ctypes.data, -1))
    if not np.array_equal(Wpub, f["W0"]):
        Wa = np.zeros((V, D))
        _lib.check(L().fm_agent_read_weights(h, Wa.ctypes.data))
        bad = np.argwhere(Wpub != f["W0"])
        raise AssertionError(f"published weights differ: {len(bad)} of {V * D} (first {bad[:3].tolist()}), "
                             f"values {Wpub.reshape(-1)[:4]} vs {np.asarray(f['W0']).reshape(-1)[:4]}; agent W "
                             f"now equal: {np.array_equal(Wa, f['W0'])}; V={V} D={D}")
    n = len(f["ids"])
    prompts, offs, seeds, want = [], [0], [], []
    for i in range(n):
        p = _dec(payload(f, int(f["prompt_off"][i])))
        prompts.append(p)
        offs.append(offs[-1] + len(p))
        sid = f"{f['ids'][i]}_{int(f['turns'][i])}_{int(f['trajs'][i])}"
        seeds.append(wl.mix_u64(wl.mix_str(wl.mix_str(wl.mix_u64(2048, 0x70CE), agent), sid), int(f["versions"][i])))
        want.append(_dec(payload(f, int(f["resp_off"][i]))))
    maxt = 256
    P = np.ascontiguousarray(np.concatenate(prompts).astype(np.int32))
    O = np.asarray(offs, np.int32)
    S = np.asarray(seeds, np.uint64)
    tok = np.zeros((n, maxt), np.int32)
    lp = np.zeros((n, maxt))
    ln = np.zeros(n, np.int32)
    try:
        _lib.check(L().fm_generate(ctx.handle, w, P.ctypes.data, O.ctypes.data, n, maxt, S.ctypes.data,
                                   tok.ctypes.data, lp.ctypes.data, ln.ctypes.data))
        for i in range(n):
            assert np.array_equal(tok[i, :ln[i]], want[i]), i
        assert ln.max() > 8 and (ln < maxt).any()  # EOS-terminated, non-trivial lengths
        assert np.all(lp[:, 0] <= 0.0)
    finally:
        L().fm_weights_destroy(w)
        L().fm_agent_destroy(h)


def test_generate_logp_matches_reference_oracle(ctx):
    from oracle import oracle as orc
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built")
    V, D = 300, 40
    rng = np.random.default_rng(4)
    W = rng.normal(size=(V, D)) * 0.5
    h = C.c_void_p()
    _lib.check(L().fm_agent_create(ctx.handle, b"g", V, D, _lib.PRECISION_PARITY_F64, C.byref(h)))
    _lib.check(L().fm_agent_set_weights(h, W.ctypes.data))
    w = C.c_void_p()
    _lib.check(L().fm_publish_weights(h, 0, C.byref(w)))
    prompts = [rng.integers(0, V, size=rng.integers(1, 7)).astype(np.int32) for _ in range(8)]
    seeds = [int(x) for x in rng.integers(0, 2 ** 62, size=8)]
    P = np.concatenate(prompts).astype(np.int32)
    O = np.cumsum([0] + [len(p) for p in prompts]).astype(np.int32)
    S = np.asarray(seeds, np.uint64)
    maxt = 64
    tok = np.zeros((8, maxt), np.int32)
    lp = np.zeros((8, maxt))
    ln = np.zeros(8, np.int32)
    try:
        _lib.check(L().fm_generate(ctx.handle, w, P.ctypes.data, O.ctypes.data, 8, maxt, S.ctypes.data,
                                   tok.ctypes.data, lp.ctypes.data, ln.ctypes.data))
        for i in range(8):
            t_ref, l_ref = orc.ref_generate(W, prompts[i], maxt, seeds[i])
            assert np.array_equal(tok[i, :ln[i]], t_ref)
            np.testing.assert_allclose(lp[i, :ln[i]], l_ref, rtol=0, atol=1e-12)
    finally:
        L().fm_weights_destroy(w)
        L().fm_agent_destroy(h)
