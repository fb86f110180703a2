"""Parity at the benchmark's full size (C2: V=32,000, D=4,096, 131M params).

The f64 oracle costs ~0.7 s per trained token at these dims, so direct
comparison uses a few tokens; a real 16 x 1,024-token micro-batch is checked
through size-independent properties of the path:
  * softmax-gradient conservation: sum_v G[t,v] = c_t (1 - sum_v p) = 0, so every
    column of the weight gradient sums to ~0 over the vocabulary;
  * linearity / GA equivalence: grad(mb1 + mb2) == grad(mb1) + grad(mb2);
  * DP partition invariance: row shards (fm_agent_set_shard) sum to the whole;
  * swap identity (checksum) of the 131M-param state.
"""
import ctypes as C

import numpy as np
import pytest

from oracle import oracle as orc
from paper_2602_09578_b200 import _lib
from paper_2602_09578_b200 import workload as wl
from paper_2602_09578_b200.engine import TrainingEngine, agent_seed, seeded_weights

pytestmark = pytest.mark.gpu
CFG = wl.CONFIGS["C2"]
V, D = CFG.vocab, CFG.feat


def rel_fro(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


@pytest.fixture(scope="module")
def c2_engine(ctx):
    eng = TrainingEngine([ctx], global_batch=64, precision=_lib.PRECISION_BF16_TC)
    eng.add_agent("agent0", V, D)
    eng.activate("agent0")
    eng.run()
    yield eng
    eng.close()


def _train(ctx, eng, samples, shard=(0, 1)):
    h = eng.handle("agent0")
    _lib.check(_lib.lib().fm_agent_set_shard(h, shard[0], shard[1]))
    arr = (_lib.fm_sample * len(samples))(*[_lib.fm_sample(ctx.put(s.prompt_payload), ctx.put(s.response_payload),
                                                           s.advantage) for s in samples])
    t = C.c_int64()
    _lib.check(_lib.lib().fm_train_micro_batch(h, arr, len(samples), 64, C.byref(t)))


def _fresh_grad(ctx, eng, batches, shard=(0, 1)):
    """Gradient accumulated over `batches` from an empty accumulator (the
    accumulator is reset by an update round trip on a throwaway copy: we
    read, then apply and restore weights)."""
    h = eng.handle("agent0")
    L = _lib.lib()
    # reset: mark accumulator empty by applying a zero-sample update is not
    # allowed (IncompleteBatch), so compute deltas instead
    before = eng.read_grad("agent0")
    for b in batches:
        _train(ctx, eng, b, shard)
    after = eng.read_grad("agent0")
    _lib.check(L.fm_agent_set_shard(h, 0, 1))
    return after - before


def _samples(step, n, L, adv_seed=0):
    s = wl.step_samples(CFG, "agent0", step, n=n, resp_len=L)
    rng = np.random.default_rng(adv_seed)
    for x in s:
        x.advantage = float(rng.normal())
    return s


def test_c2_gradient_matches_f64_oracle_few_tokens(ctx, c2_engine):
    s = _samples(0, 2, 4)
    g = _fresh_grad(ctx, c2_engine, [s])
    W0 = orc.seeded_weights(V, D, orc.agent_seed(2048, "agent0"))
    r = orc.run_agent(V, D, 2, 2, 1, [(x.prompt, x.response) for x in s], [x.advantage for x in s], W0)
    g_ref = r["last_grad"] * (2.0 / 64.0)  # oracle used G=2, the GPU G=64
    assert rel_fro(g, g_ref) <= 2e-2
    cos = float((g * g_ref).sum() / (np.linalg.norm(g) * np.linalg.norm(g_ref)))
    assert cos >= 0.999


def test_c2_full_microbatch_properties(ctx, c2_engine):
    mb1 = _samples(1, 16, 1024, adv_seed=1)
    mb2 = _samples(2, 16, 1024, adv_seed=2)
    g1 = _fresh_grad(ctx, c2_engine, [mb1])
    g2 = _fresh_grad(ctx, c2_engine, [mb2])
    g12 = _fresh_grad(ctx, c2_engine, [mb1, mb2])
    norm = np.linalg.norm(g12)
    assert norm > 0
    # conservation: column sums over the vocabulary vanish relative to the
    # column L1 mass (a kernel dropping the delta or the softmax term gives ~0.5)
    col_sum = np.abs(g12.sum(axis=0))
    col_l1 = np.abs(g12).sum(axis=0)
    live = col_l1 > 0
    assert live.mean() > 0.9
    assert np.median(col_sum[live] / col_l1[live]) < 1e-2
    # linearity (fp32 accumulation of the same bf16 partial products)
    assert rel_fro(g12, g1 + g2) < 1e-5
    # DP partition invariance: 2 row shards == whole micro-batch
    s0 = _fresh_grad(ctx, c2_engine, [mb1], shard=(0, 2))
    s1 = _fresh_grad(ctx, c2_engine, [mb1], shard=(1, 2))
    assert rel_fro(s0 + s1, g1) < 1e-5


@pytest.mark.parametrize("tier", [_lib.TIER_DEVICE, _lib.TIER_HOST])
def test_c2_swap_identity(ctx, c2_engine, tier):
    c2_engine.park_tier = tier
    before = c2_engine.checksum("agent0")
    c2_engine.suspend("agent0")
    c2_engine.activate("agent0")
    c2_engine.run()
    assert c2_engine.checksum("agent0") == before


def _host_gb():
    try:
        import psutil
        return psutil.virtual_memory().available / 2**30
    except Exception:
        return 0.0


@pytest.mark.parametrize("cfg_name", ["C3", "C5"])
def test_large_policy_gradient_matches_sparse_f64_oracle(ctx, cfg_name):
    """1.05B-parameter policies (C3: V=32,000 D=32,768; C5: V=128,000 D=8,192):
    a 2-sample x 4-token micro-batch through the tensor-core path against the
    column-sparse f64 oracle (fmo_sparse_grad, pinned bit-for-bit to the dense
    oracle in tests/test_oracle.py).  The touched feature columns match within
    the BF16_TC contract and the micro-batch grad norm — the norm of the WHOLE
    V x D gradient — matches the oracle's, so no mass lands in other columns."""
    if _host_gb() < 40:
        pytest.skip("needs ~40 GB of free host memory (seeded 1.05B-param init)")
    cfg = wl.CONFIGS[cfg_name]
    Vb, Db = cfg.vocab, cfg.feat
    s = wl.step_samples(cfg, "agent0", 0, n=2, resp_len=4)
    rng = np.random.default_rng(7)
    for x in s:
        x.advantage = float(rng.normal())
    eng = TrainingEngine([ctx], global_batch=64, precision=_lib.PRECISION_BF16_TC)
    try:
        eng.add_agent("agent0", Vb, Db)
        eng.activate("agent0")
        eng.run()
        h = eng.handle("agent0")
        arr = (_lib.fm_sample * len(s))(*[_lib.fm_sample(ctx.put(x.prompt_payload), ctx.put(x.response_payload),
                                                         x.advantage) for x in s])
        t = C.c_int64()
        _lib.check(_lib.lib().fm_train_micro_batch(h, arr, len(s), 64, C.byref(t)))
        ref = orc.sparse_grad(Vb, Db, orc.agent_seed(2048, "agent0"), [(x.prompt, x.response) for x in s],
                              [x.advantage for x in s], 64)
        cols = ref["cols"]
        g = np.empty(Vb * len(cols), dtype=np.float64)
        _lib.check(_lib.lib().fm_agent_read_grad_cols(h, cols.ctypes.data, len(cols), g.ctypes.data))
        g = g.reshape(Vb, len(cols))
        assert rel_fro(g, ref["grad"]) <= 2e-2
        cos = float((g * ref["grad"]).sum() / (np.linalg.norm(g) * np.linalg.norm(ref["grad"])))
        assert cos >= 0.999
        # whole-gradient norm (GEMM2 epilogue sum of squares) vs the oracle's
        _lib.check(_lib.lib().fm_agent_sync(h))
        rep = _lib.fm_report()
        assert _lib.lib().fm_agent_poll_report(h, t.value, C.byref(rep)) == 1
        assert abs(rep.grad_norm - ref["mb_grad_norm"]) <= 2e-2 * ref["mb_grad_norm"]
    finally:
        eng.close()
