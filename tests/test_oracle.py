"""Pins the C restatement (oracle/flexmarl_oracle.c) to the compiled reference.

Golden fixtures come from tests/golden/make_golden.py (oracle/_ref, the
unmodified reference headers).  Live cross-checks run when _ref is built.
Also covers the SPEC.md known-answer tests of the path.
"""
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as orc

G = Path(__file__).resolve().parent / "golden"


def _ld(name):
    return np.load(G / name, allow_pickle=False)


def test_rng_streams_bit_exact():
    f = _ld("rng.npz")
    for kind, name in ((0, "u64"), (1, "unit"), (2, "normal"), (3, "below")):
        for i, s in enumerate(f["seeds"]):
            buf = np.zeros(64, dtype=f[name].dtype)
            orc.olib().fmo_rng_draw(int(s), kind, 1000, 64, buf.ctypes.data)
            assert np.array_equal(buf, f[name][i]), (name, s)
    for a, s in zip(f["agent_names"], f["agent_seeds"]):
        assert orc.agent_seed(2048, str(a)) == int(s)
    assert orc.olib().fmo_mix_u64(2048, 0x5EED) == int(f["mix_u64"][0])
    assert orc.olib().fmo_mix_str(2048, b"q00001") == int(f["mix_str"][0])


def test_seeded_weights_bit_exact():
    f = _ld("rng.npz")
    for a in ("planner", "executor"):
        w = orc.seeded_weights(32, 16, orc.agent_seed(2048, a))
        assert np.array_equal(w, f[f"W0_{a}"])


def test_group_advantages_bit_exact_and_kats():
    f = _ld("adv_adam.npz")
    off = f["seg_off"]
    for i in range(len(off) - 1):
        r = f["rewards"][off[i]:off[i + 1]]
        assert np.array_equal(orc.group_advantages(r), f["adv"][off[i]:off[i + 1]])
    # [1,0,1,0] -> [1,-1,1,-1] (exact with eps: +-0.99999998000000034)
    a = orc.group_advantages([1, 0, 1, 0])
    assert np.allclose(a, [1, -1, 1, -1], atol=1e-7)
    assert a[0] == 0.99999998000000034
    # all-equal rewards -> zero advantages
    assert np.all(orc.group_advantages([0.5] * 8) == 0.0)
    assert orc.group_advantages([]).size == 0


def test_adam_bit_exact_and_kats():
    f = _ld("adv_adam.npz")
    w, m, v, st = f["w0"].copy(), np.zeros(64), np.zeros(64), 0
    for k in range(3):
        w, m, v, st = orc.adam_step(w, m, v, st, f["g"][k])
        assert np.array_equal(w, f["w"][k]) and np.array_equal(m, f["m"][k]) and np.array_equal(v, f["v"][k])
    # SURVEY §0.10 probe values: step-1 dw for g=1e-3, -1e-9, 0
    w1, *_ = orc.adam_step(np.zeros(3), np.zeros(3), np.zeros(3), 0, np.array([1e-3, -1e-9, 0.0]))
    assert abs(w1[0] - (-9.9999e-07)) < 1e-11
    assert abs(w1[1] - 9.09e-08) < 1e-10
    assert w1[2] == 0.0  # SPEC.md:450 zero gradient leaves W unchanged


def test_poll_order_matches_reference():
    f = _ld("poll.npz")
    n = len(f["ids"])
    processing = np.zeros(n, np.uint8)
    ready = f["ready"].copy()
    order = []
    while True:  # repeated polls consume the canonical order (experience_store.hpp:92-114)
        got = orc.poll_select([str(s) for s in f["ids"]], f["turns"], f["trajs"], f["versions"], ready,
                              processing, int(f["current_version"]), int(f["mb"]))
        if not got:
            break
        order += got
        processing[got] = 1
    assert order == f["order"].tolist()


@pytest.mark.parametrize("name", ["c1_planner", "c1_executor", "mid_agent0"])
def test_run_agent_matches_reference(name):
    f = _ld(f"{name}.npz")
    V, D, Gb, mb, U = (int(f[k]) for k in ("V", "D", "G", "mb", "n_updates"))
    po = f["poll_order"]
    # the restatement consumes samples in the reference's poll (canonical) order
    samples = []
    for i in po:
        p = orc.olib()
        buf = f["payloads"]
        pn = int(np.frombuffer(buf[f["prompt_off"][i]:f["prompt_off"][i] + 8].tobytes(), "<u8")[0])
        rn = int(np.frombuffer(buf[f["resp_off"][i]:f["resp_off"][i] + 8].tobytes(), "<u8")[0])
        pr = np.frombuffer(buf[f["prompt_off"][i] + 8:f["prompt_off"][i] + 8 + 8 * pn].tobytes(), "<u8").astype(np.int32)
        rr = np.frombuffer(buf[f["resp_off"][i] + 8:f["resp_off"][i] + 8 + 8 * rn].tobytes(), "<u8").astype(np.int32)
        samples.append((pr, rr))
        del p
    # canonical order check: poll order == sorted (input_id, turns, traj) within each version
    for u in range(U):
        sel = [i for i in po if f["versions"][i] == u]
        keys = [(str(f["ids"][i]), int(f["turns"][i]), int(f["trajs"][i])) for i in sel]
        assert keys == sorted(keys)
    W0 = orc.seeded_weights(V, D, orc.agent_seed(2048, str(f["agent"])))
    assert np.array_equal(W0, f["W0"])
    r = orc.run_agent(V, D, Gb, mb, U, samples, f["adv"][po], W0)
    assert np.array_equal(r["W"], f["W"])
    assert np.array_equal(r["m"], f["m"]) and np.array_equal(r["v"], f["v"])
    assert np.array_equal(r["mb_grad_norm"], f["mb_grad_norm"])
    assert np.array_equal(r["upd_grad_norm"], f["upd_grad_norm"])
    dW = r["W"] - W0
    assert np.abs(dW).max() > 0  # the run actually trained


def test_ga_equivalence_partitions():
    """4x16 vs 1x64 vs 16x4 micro-batches give the same update."""
    f = _ld("c1_planner.npz")
    po = f["poll_order"][:64]
    buf = f["payloads"]

    def dec(off):
        n = int(np.frombuffer(buf[off:off + 8].tobytes(), "<u8")[0])
        return np.frombuffer(buf[off + 8:off + 8 + 8 * n].tobytes(), "<u8").astype(np.int32)

    samples = [(dec(f["prompt_off"][i]), dec(f["resp_off"][i])) for i in po]
    W0 = f["W0"]
    outs = [orc.run_agent(32, 16, 64, mb, 1, samples, f["adv"][po], W0)["W"] for mb in (64, 16, 4)]
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[1], outs[2])


def test_pack_rows_semantics():
    samples = [(np.array([5, 6], np.int32), np.array([7, 8, 9], np.int32)),
               (np.array([], np.int32), np.array([1, 2, 3, 4, 5], np.int32))]
    r = orc.pack_rows(samples, [0.5, -2.0], 64)
    assert r["action"].tolist() == [7, 8, 9, 1, 2, 3, 4, 5]
    assert r["n_ctx"].tolist() == [2, 3, 4, 0, 1, 2, 3, 4]
    assert r["ctx4"][2].tolist() == [5, 6, 7, 8]
    assert r["ctx4"][3].tolist() == [-1, -1, -1, -1]  # empty context -> phi = 0 (policy.hpp:45)
    assert r["ctx4"][7].tolist() == [1, 2, 3, 4]
    assert r["coef"][3] == 0.0
    assert r["coef"][0] == np.float32(-0.5 / (64 * 2))


@pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")
def test_live_reference_cross_check():
    """Restatement == reference on a fresh random case (not a stored fixture)."""
    L = orc.rlib()
    rng = np.random.default_rng(123)
    V, D = 48, 24
    W = rng.normal(size=(V, D))
    for _ in range(20):
        ctx = rng.integers(-5, 100, size=rng.integers(0, 7)).astype(np.int32)
        a = int(rng.integers(0, V))
        o1 = np.zeros(V * D)
        o2 = np.zeros(V * D)
        L.ref_accumulate_grad(V, D, W.ctypes.data, ctx.ctypes.data, len(ctx), a, 0.7, o1.ctypes.data)
        orc.olib().fmo_accumulate_grad(V, D, W.ctypes.data, ctx.ctypes.data, len(ctx), a, 0.7, o2.ctypes.data)
        assert np.array_equal(o1, o2)


@pytest.mark.skipif(not orc.ref_available(), reason="oracle/_ref not built")
def test_reference_state_swap_transposes_nonsquare():
    """Documents reference defect #1: PolicyState::deserialize
    reads Matrix(r.read_u64(), r.read_u64()) with unspecified argument order,
    so a V x D state comes back D x V under GCC.  The B200 swap must not (and
    does not) replicate this; fm_agent_deserialize reads rows then cols."""
    W = np.arange(6.0).reshape(3, 2)
    blob = orc.ref_serialize_state(1, 1, 0, W, W, W)
    r = orc.ref_deserialize_state(blob, 6)
    assert (r["rows"], r["cols"]) == (2, 3)


@pytest.mark.parametrize("V,D_,seed", [(300, 50, 11), (257, 64, 12), (64, 1000, 13)])
def test_sparse_grad_equals_dense_oracle(V, D_, seed):
    """The column-sparse few-token restatement (used for full-size parity at
    C3/C5, where the dense f64 oracle needs 7 x 8.4 GB) is bit-identical to the
    dense oracle's first-update gradient on the touched columns, the rest of
    the dense gradient is exactly zero, and the micro-batch norms agree.
    Covers feature collisions (tokens >= D), 1-3-token contexts and an
    action outside the vocabulary."""
    rng = np.random.default_rng(seed)
    samples = [([int(rng.integers(0, 2 * V))], [int(rng.integers(0, V)) for _ in range(5)]),
               ([int(rng.integers(0, V)) for _ in range(8)], [int(rng.integers(0, V)) for _ in range(3)] + [V + 3]),
               ([], [int(rng.integers(0, V)) for _ in range(4)])]
    adv = rng.normal(size=len(samples))
    G = len(samples)
    aseed = orc.agent_seed(2048, f"a{seed}")
    W0 = orc.seeded_weights(V, D_, aseed)
    dense = orc.run_agent(V, D_, G, G, 1, samples, adv, W0)
    sp = orc.sparse_grad(V, D_, aseed, samples, adv, G)
    g = dense["last_grad"]
    np.testing.assert_array_equal(g[:, sp["cols"]], sp["grad"])
    rest = np.ones(D_, dtype=bool)
    rest[sp["cols"]] = False
    assert not np.any(g[:, rest])
    assert sp["mb_grad_norm"] == dense["mb_grad_norm"][0]


@pytest.mark.parametrize("V,D_,mb,seed", [(64, 16, 4, 0), (300, 72, 6, 1), (1000, 256, 4, 2), (257, 40, 3, 3)])
def test_step_grad_equals_dense_oracle(V, D_, mb, seed):
    """fmo_step_grad (the full-size parity checker: threads over tokens, then
    over vocabulary blocks) is bit-identical to the dense sequential
    restatement fmo_run_agent — gradient over all V x D and every micro-batch
    grad norm — for any thread count, with empty prompts / responses, context
    collisions, negative and out-of-vocabulary tokens.  The norms sum their
    squares per vocabulary block, so they agree to rounding (1e-12), not bitwise."""
    rng = np.random.default_rng(seed)
    n = 12
    samples = [(rng.integers(-3, 3 * V, size=int(rng.integers(0, 7))).astype(np.int32),
                rng.integers(0, V + 2, size=int(rng.integers(0, 40))).astype(np.int32)) for _ in range(n)]
    adv = rng.normal(size=n)
    W0 = rng.normal(size=(V, D_)) * 0.5
    ref = orc.run_agent(V, D_, n, mb, 1, samples, adv, W0)
    for threads in (1, 3, 8):
        r = orc.step_grad(V, D_, W0.T.copy(), samples, adv, n, mb=mb, threads=threads)
        np.testing.assert_array_equal(r["gradT"].T, ref["last_grad"])
        np.testing.assert_allclose(r["mb_grad_norms"], ref["mb_grad_norm"], rtol=1e-12)
