"""GPU parity of the B200 path against the reference (golden fixtures from the
compiled reference, the C restatement, and a plain torch fp32 restatement of
the dense op for the tensor-core kernels).

Tolerances (restated):
  * selection / gather / indexing: bit-exact;
  * PARITY_F64 (fp64 SIMT): grad norms rel 1e-9, dW_step rel-Frobenius 1e-9,
    delta-W after N updates rel-Frobenius 1e-6;
  * BF16_TC (tcgen05, bf16 operands, fp32 accumulate): per-step gradient
    rel-Frobenius <= 2e-2 and cosine >= 0.999; micro-batch grad norms rel 2e-2;
    delta-W after N updates rel-Frobenius <= 5e-2 with <= 1% of elements
    differing by more than 0.5*lr*N (Adam sign flips where g ~ 0).
"""
from pathlib import Path

import ctypes as C
import numpy as np
import pytest

from oracle import oracle as orc
from paper_2602_09578_b200 import _lib
from paper_2602_09578_b200.engine import group_advantages, seeded_weights, agent_seed
from fixture_runner import run_fixture

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def _ld(name):
    return np.load(GOLD / name, allow_pickle=False)


def rel_fro(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def test_seeded_weights_native_bit_exact():
    f = _ld("rng.npz")
    for a in ("planner", "executor"):
        assert np.array_equal(seeded_weights(32, 16, agent_seed(2048, a)), f[f"W0_{a}"])
    big = seeded_weights(1000, 300, 99, threads=7)  # threaded split == sequential stream
    assert np.array_equal(big, orc.seeded_weights(1000, 300, 99))


def test_group_advantages_kernel(ctx):
    f = _ld("adv_adam.npz")
    out = group_advantages(ctx, f["rewards"], f["seg_off"])
    np.testing.assert_allclose(out, f["adv"], rtol=0, atol=1e-12 * max(1.0, np.abs(f["adv"]).max()))
    assert np.all(group_advantages(ctx, [0.5] * 8) == 0.0)


@pytest.mark.parametrize("name", ["c1_planner", "c1_executor"])
def test_parity_f64_matches_reference(ctx, name):
    f = _ld(f"{name}.npz")
    r = run_fixture(ctx, f, _lib.PRECISION_PARITY_F64)
    assert np.array_equal(r["poll_order"], f["poll_order"])  # bit-exact selection
    np.testing.assert_allclose(r["mb_grad_norm"], f["mb_grad_norm"], rtol=1e-9)
    np.testing.assert_allclose(r["upd_grad_norm"], f["upd_grad_norm"], rtol=1e-9)
    dW_ref = f["W"] - f["W0"]
    dW = r["W"] - f["W0"]
    assert rel_fro(dW, dW_ref) < 1e-6
    lr, N = 1e-6, int(f["n_updates"])
    assert np.mean(np.abs(dW - dW_ref) > 0.5 * lr * N) <= 1e-3
    # moments are stored fp32 (4 B/param): relative to the moment scale
    np.testing.assert_allclose(r["m"], f["m"], rtol=1e-6, atol=1e-6 * np.abs(f["m"]).max())
    np.testing.assert_allclose(r["v"], f["v"], rtol=1e-6, atol=1e-6 * np.abs(f["v"]).max())


def test_gather_bit_exact(ctx):
    f = _ld("c1_planner.npz")
    seen = {}

    def after_mb(eng, agent, batch):
        if "rows" in seen:
            return
        idx = [int(np.where((f["ids"] == r.sample_id.input_id) & (f["trajs"] == r.sample_id.trajectory_id)
                            & (f["versions"] == r.policy_version))[0][0]) for r in batch.samples]
        buf = f["payloads"]

        def dec(off):
            n = int(np.frombuffer(buf[off:off + 8].tobytes(), "<u8")[0])
            return np.frombuffer(buf[off + 8:off + 8 + 8 * n].tobytes(), "<u8").astype(np.uint32).view(np.int32)

        samples = [(dec(int(f["prompt_off"][i])), dec(int(f["resp_off"][i]))) for i in idx]
        want = orc.pack_rows(samples, f["adv"][idx], int(f["G"]))
        M = len(want["action"])
        got = {k: np.zeros(M, np.int32) for k in ("action", "n_ctx", "sample")}
        got["ctx4"] = np.zeros((M, 4), np.int32)
        got["coef"] = np.zeros(M, np.float32)
        _lib.check(_lib.lib().fm_debug_read_rows(ctx.handle, M, got["action"].ctypes.data,
                                                 got["ctx4"].ctypes.data, got["n_ctx"].ctypes.data,
                                                 got["sample"].ctypes.data, got["coef"].ctypes.data))
        seen["rows"] = (want, got)

    run_fixture(ctx, f, _lib.PRECISION_PARITY_F64, hooks={"after_mb": after_mb})
    want, got = seen["rows"]
    for k in ("action", "ctx4", "n_ctx", "sample"):
        assert np.array_equal(got[k], want[k]), k
    assert np.array_equal(got["coef"].view(np.uint32), want["coef"].view(np.uint32))


def _oracle_grad_step0(f):
    """-(1/G) sum term of update 0 (f64), from the restatement."""
    po = f["poll_order"]
    buf = f["payloads"]

    def dec(off):
        n = int(np.frombuffer(buf[off:off + 8].tobytes(), "<u8")[0])
        return np.frombuffer(buf[off + 8:off + 8 + 8 * n].tobytes(), "<u8").astype(np.uint32).view(np.int32)

    G = int(f["G"])
    sel = po[:G]
    samples = [(dec(int(f["prompt_off"][i])), dec(int(f["resp_off"][i]))) for i in sel]
    r = orc.run_agent(int(f["V"]), int(f["D"]), G, int(f["mb"]), 1, samples, f["adv"][sel], f["W0"])
    return r["last_grad"]


def test_tensor_core_path_matches_reference(ctx):
    f = _ld("mid_agent0.npz")
    r = run_fixture(ctx, f, _lib.PRECISION_BF16_TC)
    assert np.array_equal(r["poll_order"], f["poll_order"])
    g_ref = _oracle_grad_step0(f)
    g = r["grads"][0]
    assert rel_fro(g, g_ref) <= 2e-2
    cos = float((g * g_ref).sum() / (np.linalg.norm(g) * np.linalg.norm(g_ref)))
    assert cos >= 0.999
    np.testing.assert_allclose(r["mb_grad_norm"], f["mb_grad_norm"], rtol=2e-2)
    np.testing.assert_allclose(r["upd_grad_norm"], f["upd_grad_norm"], rtol=2e-2)
    dW_ref = f["W"] - f["W0"]
    dW = r["W"] - f["W0"]
    assert rel_fro(dW, dW_ref) <= 5e-2
    assert np.mean(np.abs(dW - dW_ref) > 0.5 * 1e-6 * int(f["n_updates"])) <= 1e-2


def test_tensor_core_kernels_vs_torch_fp32(ctx):
    """One micro-batch through K-gather/K-pos/K-stats/K-lse/K-band/K-GEMM2
    against a plain torch fp32 restatement of the same dense op on the same
    bf16-rounded operands (V=1000 exercises the N-tile tail)."""
    import torch
    from paper_2602_09578_b200.engine import TrainingEngine
    V, D, L, n = 1000, 136, 200, 16
    rng = np.random.default_rng(5)
    W0 = rng.normal(size=(V, D)) * 0.5
    samples = [(rng.integers(0, V, size=rng.integers(0, 6)).astype(np.int32),
                rng.integers(0, V, size=L).astype(np.int32)) for _ in range(n)]
    adv = rng.normal(size=n)
    ctx.reset_arena()
    eng = TrainingEngine([ctx], global_batch=64, precision=_lib.PRECISION_BF16_TC)
    eng.add_agent("t", V, D)
    eng.activate("t")
    _lib.check(_lib.lib().fm_agent_set_weights(eng.handle("t"), np.ascontiguousarray(W0).ctypes.data))
    arr = (_lib.fm_sample * n)(*[_lib.fm_sample(ctx.put(orc.encode(p)), ctx.put(orc.encode(r)), a)
                                 for (p, r), a in zip(samples, adv)])
    t = C.c_int64()
    _lib.check(_lib.lib().fm_train_micro_batch(eng.handle("t"), arr, n, 64, C.byref(t)))
    g = eng.read_grad("t")
    M = n * L
    logp = np.zeros(M)
    _lib.check(_lib.lib().fm_agent_read_logp(eng.handle("t"), logp.ctypes.data, M))
    eng.close()
    # torch fp32 restatement of the dense formulation
    rows = orc.pack_rows(samples, adv, 64)
    phi = torch.zeros(M, D, dtype=torch.float32, device="cuda")
    for j in range(4):
        valid = rows["n_ctx"] > j
        r_idx = torch.tensor(np.nonzero(valid)[0], device="cuda")
        f_idx = torch.tensor((rows["ctx4"][valid, j].astype(np.int64) % D), device="cuda")
        phi.index_put_((r_idx, f_idx), torch.ones(len(r_idx), device="cuda"), accumulate=True)
    w16 = torch.tensor(W0, device="cuda").to(torch.bfloat16).float()
    nctx = torch.tensor(rows["n_ctx"], device="cuda").float()
    rs = torch.where(nctx > 0, 1.0 / nctx.clamp(min=1), torch.zeros_like(nctx))
    z = (phi @ w16.T) * rs[:, None]
    lse = torch.logsumexp(z, dim=1)
    act = torch.tensor(rows["action"].astype(np.int64), device="cuda")
    lp_t = (z.gather(1, act[:, None])[:, 0] - lse).cpu().numpy()
    p = torch.softmax(z, dim=1)
    coef = torch.tensor(rows["coef"], device="cuda")
    Gm = -p
    Gm[torch.arange(M, device="cuda"), act] += 1.0
    Gm = Gm * coef[:, None]
    g_t = (Gm.T @ phi).double().cpu().numpy()
    np.testing.assert_allclose(logp, lp_t, atol=2e-3)
    assert rel_fro(g, g_t) < 1e-2


@pytest.mark.parametrize("tier", [_lib.TIER_HOST, _lib.TIER_DEVICE])
def test_swap_identity(ctx, tier):
    """suspend -> activate is the identity on the training state,
    including a mid-step gradient accumulator."""
    from paper_2602_09578_b200.engine import TrainingEngine
    f = _ld("mid_agent0.npz")
    V, D = int(f["V"]), int(f["D"])
    ctx.reset_arena()
    eng = TrainingEngine([ctx], global_batch=64, precision=_lib.PRECISION_BF16_TC, park_tier=tier)
    eng.add_agent("s", V, D)
    eng.activate("s")
    buf = f["payloads"]
    arr = (_lib.fm_sample * 16)(*[_lib.fm_sample(ctx.put(buf[int(f["prompt_off"][i]):].tobytes()[:8 + 8 * int(
        np.frombuffer(buf[int(f["prompt_off"][i]):int(f["prompt_off"][i]) + 8].tobytes(), "<u8")[0])]),
        ctx.put(buf[int(f["resp_off"][i]):].tobytes()[:8 + 8 * int(
            np.frombuffer(buf[int(f["resp_off"][i]):int(f["resp_off"][i]) + 8].tobytes(), "<u8")[0])]),
        float(f["adv"][i])) for i in range(16)])
    t = C.c_int64()
    _lib.check(_lib.lib().fm_train_micro_batch(eng.handle("s"), arr, 16, 64, C.byref(t)))
    before = eng.checksum("s")
    g_before = eng.read_grad("s")
    eng.suspend("s")
    eng.activate("s")
    eng.run()
    assert eng.checksum("s") == before
    assert np.array_equal(eng.read_grad("s"), g_before)
    eng.close()


def test_e2e_host_path_equals_arena_path(ctx):
    from paper_2602_09578_b200.engine import TrainingEngine
    rng = np.random.default_rng(9)
    V, D, n = 512, 64, 8
    samples = [(rng.integers(0, V, 5).astype(np.int32), rng.integers(0, V, 100).astype(np.int32)) for _ in range(n)]
    adv = rng.normal(size=n)
    grads = []
    for host in (False, True):
        ctx.reset_arena()
        eng = TrainingEngine([ctx], global_batch=64, precision=_lib.PRECISION_BF16_TC)
        eng.add_agent("e", V, D)
        eng.activate("e")
        t = C.c_int64()
        if host:
            keep = [(orc.encode(p), orc.encode(r)) for p, r in samples]
            bufs = [(C.create_string_buffer(a, len(a)), C.create_string_buffer(b, len(b))) for a, b in keep]
            arr = (_lib.fm_host_sample * n)(*[_lib.fm_host_sample(C.cast(a, C.c_void_p), C.cast(b, C.c_void_p), x)
                                              for (a, b), x in zip(bufs, adv)])
            _lib.check(_lib.lib().fm_train_micro_batch_host(eng.handle("e"), arr, n, 64, C.byref(t)))
        else:
            arr = (_lib.fm_sample * n)(*[_lib.fm_sample(ctx.put(orc.encode(p)), ctx.put(orc.encode(r)), x)
                                         for (p, r), x in zip(samples, adv)])
            _lib.check(_lib.lib().fm_train_micro_batch(eng.handle("e"), arr, n, 64, C.byref(t)))
        grads.append(eng.read_grad("e"))
        eng.close()
    assert np.array_equal(grads[0], grads[1])


def test_incomplete_batch_and_inactive_errors(ctx):
    from paper_2602_09578_b200.engine import TrainingEngine, MarlsimError
    eng = TrainingEngine([ctx], global_batch=64, precision=_lib.PRECISION_BF16_TC)
    eng.add_agent("x", 256, 64)
    with pytest.raises(MarlsimError) as e:
        eng.apply_global_update("x")
    assert e.value.name == "InactiveGroup"
    eng.activate("x")
    with pytest.raises(MarlsimError) as e:
        eng.apply_global_update("x")
    assert e.value.name == "IncompleteBatch"
    eng.close()


@pytest.mark.parametrize("V,D", [(1000, 136), (300, 72), (4000, 4096)])
def test_w16t_shadow_tracks_weights(ctx, V, D):
    """The transposed bf16 shadow W16^T (the rows K-stats / K-band stream) is
    bf16(W) after every writer: set_weights (K-w16t), the Adam step (the
    tile-transposed store fused into K-adam), update-and-park + activate (the
    parked copy), and a host-tier swap (regenerated from W).  Read back through
    the bf16 weight publish, which untransposes it."""
    import torch
    from paper_2602_09578_b200.engine import TrainingEngine
    L = _lib.lib()
    rng = np.random.default_rng(V)
    W0 = rng.normal(size=(V, D)) * 0.5
    eng = TrainingEngine([ctx], global_batch=16, precision=_lib.PRECISION_BF16_TC)

    def check_shadow(h, tag=""):
        W = np.empty(V * D)
        _lib.check(L.fm_agent_read_weights(h, W.ctypes.data))
        w = C.c_void_p()
        _lib.check(L.fm_publish_weights(h, 2, C.byref(w)))
        out = torch.empty(V * D, dtype=torch.bfloat16)
        _lib.check(L.fm_weights_get(w, out.data_ptr(), -1))
        _lib.check(L.fm_weights_destroy(w))
        want = torch.tensor(W).float().bfloat16()
        bad = (out.view(torch.int16) != want.view(torch.int16)).reshape(V, D)
        if bad.any():
            idx = bad.nonzero()
            raise AssertionError(f"{tag}: {int(bad.sum())} shadow elements differ; vocab rows "
                                 f"{idx[:, 0].min().item()}..{idx[:, 0].max().item()}, features "
                                 f"{idx[:, 1].min().item()}..{idx[:, 1].max().item()}")

    try:
        eng.add_agent("t", V, D)
        eng.activate("t")
        eng.run()
        h = eng.handle("t")
        _lib.check(L.fm_agent_set_weights(h, np.ascontiguousarray(W0).ctypes.data))
        check_shadow(h, "set_weights")
        samples = [(rng.integers(0, V, size=4).astype(np.int32), rng.integers(0, V, size=20).astype(np.int32))
                   for _ in range(16)]
        arr = (_lib.fm_sample * 16)(*[_lib.fm_sample(ctx.put(orc.encode(p)), ctx.put(orc.encode(r)), a)
                                      for (p, r), a in zip(samples, rng.normal(size=16))])
        t = C.c_int64()
        for step in range(3):
            _lib.check(L.fm_train_micro_batch(h, arr, 16, 16, C.byref(t)))
            if step == 1:
                _lib.check(L.fm_apply_update_park(h, 16, 1e-2, 0.9, 0.999, 1e-8, None, None))
                _lib.check(L.fm_agent_activate(h, ctx.handle))
            else:
                _lib.check(L.fm_apply_update(h, 16, 1e-2, 0.9, 0.999, 1e-8, None, None))
            check_shadow(h, f"step {step}")
        _lib.check(L.fm_agent_suspend(h, _lib.TIER_HOST, -1))
        _lib.check(L.fm_agent_activate(h, ctx.handle))
        check_shadow(h, "host-tier swap")
    finally:
        eng.close()


def test_destroy_with_unconsumed_swap_in(ctx):
    """Destroying an agent whose swap-in (activate prefetch) was never consumed
    must not hand its training slot to the next agent while the copy-in is
    still writing into it (regression: the next agent's weights were clobbered)."""
    L = _lib.lib()
    V, D = 2000, 512
    for _ in range(3):
        h = C.c_void_p()
        _lib.check(L.fm_agent_create(ctx.handle, b"victim", V, D, _lib.PRECISION_BF16_TC, C.byref(h)))
        Wc = np.full(V * D, 0.25)
        _lib.check(L.fm_agent_set_weights(h, Wc.ctypes.data))
        _lib.check(L.fm_agent_suspend(h, _lib.TIER_HOST, -1))
        _lib.check(L.fm_agent_activate(h, ctx.handle))  # PCIe copy-in in flight
        _lib.check(L.fm_agent_destroy(h))
        g = C.c_void_p()
        _lib.check(L.fm_agent_create(ctx.handle, b"next", V, D, _lib.PRECISION_BF16_TC, C.byref(g)))
        W = np.random.default_rng(3).normal(size=V * D)
        _lib.check(L.fm_agent_set_weights(g, W.ctypes.data))
        out = np.zeros(V * D)
        _lib.check(L.fm_agent_read_weights(g, out.ctypes.data))
        _lib.check(L.fm_agent_destroy(g))
        assert np.array_equal(out, W)


def test_ppo_clip_surrogate_vs_torch_fp32(ctx):
    """Optional PPO clipped-ratio surrogate (a8): the gradient flows, scaled by
    rho = exp(logp - old_logp), only through rows whose unclipped branch is the
    min (A >= 0: rho <= 1+eps; A < 0: rho >= 1-eps).  Checked against a torch
    fp32 restatement; target ratios stay 0.1 away from the clip edges so bf16
    logits cannot flip a row's branch."""
    import torch
    from paper_2602_09578_b200.engine import TrainingEngine
    V, D, L_, n, eps = 1000, 136, 120, 16, 0.2
    rng = np.random.default_rng(21)
    W0 = rng.normal(size=(V, D)) * 0.5
    samples = [(rng.integers(0, V, size=rng.integers(1, 6)).astype(np.int32),
                rng.integers(0, V, size=L_).astype(np.int32)) for _ in range(n)]
    adv = rng.normal(size=n)
    rows = orc.pack_rows(samples, adv, 64)
    M = n * L_
    # torch fp32 restatement of the dense op on the bf16 shadow
    phi = torch.zeros(M, D, dtype=torch.float32, device="cuda")
    for j in range(4):
        valid = rows["n_ctx"] > j
        r_idx = torch.tensor(np.nonzero(valid)[0], device="cuda")
        f_idx = torch.tensor((rows["ctx4"][valid, j].astype(np.int64) % D), device="cuda")
        phi.index_put_((r_idx, f_idx), torch.ones(len(r_idx), device="cuda"), accumulate=True)
    w16 = torch.tensor(W0, device="cuda").float().to(torch.bfloat16).float()
    nctx = torch.tensor(rows["n_ctx"], device="cuda").float()
    rs = torch.where(nctx > 0, 1.0 / nctx.clamp(min=1), torch.zeros_like(nctx))
    z = (phi @ w16.T) * rs[:, None]
    lse = torch.logsumexp(z, dim=1)
    act = torch.tensor(rows["action"].astype(np.int64), device="cuda")
    lp = z.gather(1, act[:, None])[:, 0] - lse
    rho_t = torch.tensor(rng.choice([0.5, 0.7, 1.0, 1.3, 1.6], size=M), device="cuda").float()
    old = (lp - torch.log(rho_t)).cpu().numpy().astype(np.float32)
    a_row = torch.tensor(adv[rows["sample"]], device="cuda").float()
    active = torch.where(a_row >= 0, rho_t <= 1 + eps, rho_t >= 1 - eps)
    coef = torch.tensor(rows["coef"], device="cuda") * torch.where(active, rho_t, torch.zeros_like(rho_t))
    p = torch.softmax(z, dim=1)
    Gm = -p
    Gm[torch.arange(M, device="cuda"), act] += 1.0
    g_t = ((Gm * coef[:, None]).T @ phi).double().cpu().numpy()
    assert 0.2 < float(active.float().mean()) < 0.95  # both branches exercised
    # the same micro-batch through the tensor-core path with the clip enabled
    ctx.reset_arena()
    eng = TrainingEngine([ctx], global_batch=64, precision=_lib.PRECISION_BF16_TC)
    eng.add_agent("c", V, D)
    eng.activate("c")
    h = eng.handle("c")
    L = _lib.lib()
    _lib.check(L.fm_agent_set_weights(h, W0.ctypes.data))
    _lib.check(L.fm_agent_set_clip(h, eps, old.ctypes.data, M))
    arr = (_lib.fm_sample * n)(*[_lib.fm_sample(ctx.put(orc.encode(pr)), ctx.put(orc.encode(r)), a)
                                 for (pr, r), a in zip(samples, adv)])
    t = C.c_int64()
    _lib.check(L.fm_train_micro_batch(h, arr, n, 64, C.byref(t)))
    g = eng.read_grad("c")
    eng.close()
    assert rel_fro(g, g_t) < 1e-2


def _train_one(ctx, V, D_, samples, adv, G=64):
    from paper_2602_09578_b200.engine import TrainingEngine
    eng = TrainingEngine([ctx], global_batch=G, precision=_lib.PRECISION_BF16_TC)
    try:
        eng.add_agent("sk", V, D_)
        eng.activate("sk")
        eng.run()
        h = eng.handle("sk")
        arr = (_lib.fm_sample * len(samples))(*[_lib.fm_sample(ctx.put(orc.encode(p)), ctx.put(orc.encode(r)), a)
                                                for (p, r), a in zip(samples, adv)])
        t = C.c_int64()
        _lib.check(_lib.lib().fm_train_micro_batch(h, arr, len(samples), G, C.byref(t)))
        _lib.check(_lib.lib().fm_agent_sync(h))
        rep = _lib.fm_report()
        assert _lib.lib().fm_agent_poll_report(h, t.value, C.byref(rep)) == 1
        return eng.read_grad("sk"), rep.grad_norm
    finally:
        eng.close()


@pytest.mark.parametrize("V,D_,resp", [(256 * 75, 256, 6), (256 * 80, 512, 40), (256 * 150, 256, 3)])
def test_gemm2_partial_waves(ctx, V, D_, resp):
    """K-GEMM2 tile counts that leave a partial last wave on 74 CTA pairs (75,
    160 and 150 output tiles, 1-2 K iterations per segment) against the f64
    oracle within the BF16_TC contract, micro-batch grad norm included."""
    rng = np.random.default_rng(V + D_)
    samples = [([int(x) for x in rng.integers(0, V, size=8)], [int(x) for x in rng.integers(0, V, size=resp)])
               for _ in range(16)]
    adv = rng.normal(size=16)
    g, n = _train_one(ctx, V, D_, samples, adv)
    assert np.linalg.norm(g) > 0
    ref = orc.sparse_grad(V, D_, agent_seed(2048, "sk"), samples, adv, 64)
    assert rel_fro(g[:, ref["cols"]], ref["grad"]) <= 2e-2
    assert abs(n - ref["mb_grad_norm"]) <= 2e-2 * ref["mb_grad_norm"]
    # columns no context touches stay exactly zero
    untouched = np.setdiff1d(np.arange(D_), ref["cols"])
    assert not np.any(g[:, untouched])


def test_update_park_equals_update_then_suspend(ctx):
    """fm_apply_update_park (K-adam writes W/m/v/W16^T straight into the
    parking buffer) == fm_apply_update + fm_agent_suspend(device): after
    re-activation the state checksums (W, m, v, W16), weights, moments and the
    next step's gradient are bit-identical, and equal the resident run's."""
    from paper_2602_09578_b200.engine import TrainingEngine
    L = _lib.lib()
    V, D_ = 2048, 256
    rng = np.random.default_rng(5)
    batches = [[([int(x) for x in rng.integers(0, V, size=8)], [int(x) for x in rng.integers(0, V, size=12)])
                for _ in range(16)] for _ in range(8)]
    adv = [rng.normal(size=16) for _ in range(8)]

    def run(mode):
        eng = TrainingEngine([ctx], global_batch=64, precision=_lib.PRECISION_BF16_TC)
        try:
            eng.add_agent("p", V, D_)
            eng.activate("p")
            eng.run()
            h = eng.handle("p")
            for step in range(2):
                for b in range(4):
                    k = step * 4 + b
                    arr = (_lib.fm_sample * 16)(*[_lib.fm_sample(ctx.put(orc.encode(p)), ctx.put(orc.encode(r)), a)
                                                  for (p, r), a in zip(batches[k], adv[k])])
                    t = C.c_int64()
                    _lib.check(L.fm_train_micro_batch(h, arr, 16, 64, C.byref(t)))
                if mode == "park" and step == 0:
                    _lib.check(L.fm_apply_update_park(h, 64, 1e-3, 0.9, 0.999, 1e-8, None, None))
                    assert L.fm_agent_is_active(h) == 0
                else:
                    _lib.check(L.fm_apply_update(h, 64, 1e-3, 0.9, 0.999, 1e-8, None, None))
                    if mode == "copy" and step == 0:
                        _lib.check(L.fm_agent_suspend(h, _lib.TIER_DEVICE, -1))
                if mode != "resident" and step == 0:
                    _lib.check(L.fm_agent_activate(h, ctx.handle))
            cs = C.c_uint64()
            _lib.check(L.fm_agent_state_checksum(h, C.byref(cs)))
            W = np.empty(V * D_, dtype=np.float64)
            _lib.check(L.fm_agent_read_weights(h, W.ctypes.data))
            return cs.value, W
        finally:
            eng.close()

    park, copy, res = run("park"), run("copy"), run("resident")
    assert park[0] == copy[0] == res[0]
    np.testing.assert_array_equal(park[1], res[1])
    assert np.any(park[1] != seeded_weights(V, D_, agent_seed(2048, "p")).reshape(-1))


def test_update_park_and_read_cols_error_paths(ctx):
    """fm_apply_update_park keeps the reference's update errors (IncompleteBatch
    before anything changes) and refuses a parity-mode agent; the agent stays
    active and usable after a refused call.  fm_agent_read_grad_cols rejects
    out-of-range columns."""
    from paper_2602_09578_b200.engine import TrainingEngine
    L = _lib.lib()
    eng = TrainingEngine([ctx], global_batch=64, precision=_lib.PRECISION_PARITY_F64)
    try:
        eng.add_agent("e", 64, 16)
        eng.activate("e")
        eng.run()
        h = eng.handle("e")
        assert L.fm_apply_update_park(h, 64, 1e-3, 0.9, 0.999, 1e-8, None, None) == 25  # IncompleteBatch
        arr = (_lib.fm_sample * 64)(*[_lib.fm_sample(ctx.put(orc.encode([1, 2, 3])), ctx.put(orc.encode([4, 5])), 0.5)
                                      for _ in range(64)])
        t = C.c_int64()
        _lib.check(L.fm_train_micro_batch(h, arr, 64, 64, C.byref(t)))
        assert L.fm_apply_update_park(h, 64, 1e-3, 0.9, 0.999, 1e-8, None, None) == _lib.FM_ERR_INVALID_ARG
        assert L.fm_agent_is_active(h) == 1
        cols = np.array([0, 16], dtype=np.int64)
        out = np.zeros(64 * 2)
        assert L.fm_agent_read_grad_cols(h, cols.ctypes.data, 2, out.ctypes.data) == _lib.FM_ERR_INVALID_ARG
        _lib.check(L.fm_apply_update(h, 64, 1e-3, 0.9, 0.999, 1e-8, None, None))
    finally:
        eng.close()


@pytest.mark.parametrize("a_mn,b_mn", [(0, 0), (1, 0), (0, 1), (1, 1)])
@pytest.mark.parametrize("M,N,K", [(512, 512, 256), (384, 768, 448)])
def test_tcgen05_gemm_operand_majorness(ctx, a_mn, b_mn, M, N, K):
    """The CTA-pair tcgen05 GEMM with K-major ([M][K] / [N][K]) or MN-major
    ([K][M] / [K][N]) bf16 operands (SWIZZLE_128B smem descriptors) against a
    torch fp32 product of the same bf16 values."""
    import torch
    g = torch.Generator(device="cuda").manual_seed(M + N + K + 2 * a_mn + b_mn)
    a = torch.randn(M, K, device="cuda", generator=g).bfloat16()
    b = torch.randn(N, K, device="cuda", generator=g).bfloat16()
    A = a.t().contiguous() if a_mn else a
    B = b.t().contiguous() if b_mn else b
    C_ = torch.empty(M, N, device="cuda", dtype=torch.float32)
    _lib.check(_lib.lib().fm_debug_gemm(ctx.handle, A.data_ptr(), B.data_ptr(), a_mn, b_mn, M, N, K, C_.data_ptr()))
    ref = a.float() @ b.float().t()
    err = (C_ - ref).norm() / ref.norm()
    assert float(err) < 1e-5


def test_gemm2_rows_counter(ctx):
    """fm_ctx_gemm2_rows: K-GEMM2's executed K rows (the bench's executed-flop
    roofline) — every 256-feature block's segment is padded to a multiple of 64
    rows (at least 64), and every context position with a token has one row."""
    f = _ld("mid_agent0.npz")
    L = _lib.lib()
    rows = C.c_int64()
    _lib.check(L.fm_ctx_gemm2_rows(ctx.handle, C.byref(rows), 1))
    r = run_fixture(ctx, f, _lib.PRECISION_BF16_TC)
    _lib.check(L.fm_ctx_gemm2_rows(ctx.handle, C.byref(rows), 1))
    n_mb = len(r["mb_grad_norm"])
    nblk = (int(f["D"]) + 255) // 256
    assert rows.value % 64 == 0 and rows.value >= 64 * nblk * n_mb


@pytest.mark.parametrize("V,D_,n_samples,resp", [(300, 200, 5, 7), (1000, 520, 16, 33), (4100, 96, 3, 2),
                                                 (520, 1000, 16, 64), (2056, 72, 40, 1)])
def test_band_pipeline_odd_shapes(ctx, V, D_, n_samples, resp):
    """The band pipeline on ragged shapes — V and D not multiples of 256 (partial
    last vocabulary slice / feature block), V not a multiple of 8 (W16^T row
    padding), blocks no position touches, positions whose features share a
    block, prompts shorter than the 4-token window (missing positions),
    one-token responses (a sample's positions end before its 4th), tiny
    micro-batches — against the column-sparse f64 oracle."""
    rng = np.random.default_rng(V * 7 + D_)
    samples = [([int(x) for x in rng.integers(0, 3 * V, size=int(rng.integers(0, 6)))],
                [int(x) for x in rng.integers(0, V, size=resp)]) for _ in range(n_samples)]
    adv = rng.normal(size=n_samples)
    g, n = _train_one(ctx, V, D_, samples, adv)
    ref = orc.sparse_grad(V, D_, agent_seed(2048, "sk"), samples, adv, 64)
    assert rel_fro(g[:, ref["cols"]], ref["grad"]) <= 2e-2
    assert abs(n - ref["mb_grad_norm"]) <= 2e-2 * ref["mb_grad_norm"]
    untouched = np.setdiff1d(np.arange(D_), ref["cols"])
    assert not np.any(g[:, untouched])


@pytest.mark.parametrize("nranks", [2, 3, 5])
def test_shard_gradients_sum_to_whole(ctx, nranks):
    """Token-balanced DP shards (fm_agent_set_shard): each rank's row range cuts
    samples mid-sequence, so context positions at a cut get partial gradient
    rows on both sides; the shards' gradients add up to the unsharded one (fp32
    summation order), on one GPU."""
    from paper_2602_09578_b200.engine import TrainingEngine
    V, D_ = 1000, 136
    rng = np.random.default_rng(nranks)
    samples = [([int(x) for x in rng.integers(0, V, size=int(rng.integers(1, 7)))],
                [int(x) for x in rng.integers(0, V, size=int(rng.integers(1, 90)))]) for _ in range(16)]
    adv = rng.normal(size=16)
    whole, _ = _train_one(ctx, V, D_, samples, adv)
    total = np.zeros_like(whole)
    L = _lib.lib()
    for r in range(nranks):
        eng = TrainingEngine([ctx], global_batch=64, precision=_lib.PRECISION_BF16_TC)
        try:
            eng.add_agent("sk", V, D_)
            eng.activate("sk")
            eng.run()
            h = eng.handle("sk")
            _lib.check(L.fm_agent_set_shard(h, r, nranks))
            arr = (_lib.fm_sample * 16)(*[_lib.fm_sample(ctx.put(orc.encode(p)), ctx.put(orc.encode(q)), a)
                                          for (p, q), a in zip(samples, adv)])
            t = C.c_int64()
            _lib.check(L.fm_train_micro_batch(h, arr, 16, 64, C.byref(t)))
            total += eng.read_grad("sk")
        finally:
            eng.close()
    # positions at a cut are rounded to bf16 as two partial rows instead of one sum
    assert rel_fro(total, whole) <= 1e-3


def test_segment_buffer_reuse_across_widths(ctx):
    """K-GEMM2's A' segments are one workspace reused by agents of every width:
    an agent whose V is not a multiple of 8 leaves its rows' pitch columns
    behind, and a later, wider agent's segment padding rows (B' = 0 there) read
    them.  They must be finite — 0 x NaN would poison that agent's dW (the
    regression: K-band stored arithmetic on stale ring bytes past V)."""
    L = _lib.lib()
    rng = np.random.default_rng(17)
    for V, D in [(300, 72), (1004, 136), (4000, 4096)]:
        h = C.c_void_p()
        _lib.check(L.fm_agent_create(ctx.handle, b"w", V, D, _lib.PRECISION_BF16_TC, C.byref(h)))
        try:
            W0 = np.ascontiguousarray(rng.normal(size=(V, D)) * 0.5)
            _lib.check(L.fm_agent_set_weights(h, W0.ctypes.data))
            arr = (_lib.fm_sample * 16)(*[_lib.fm_sample(ctx.put(orc.encode(rng.integers(0, V, size=4).astype(np.int32))),
                                                         ctx.put(orc.encode(rng.integers(0, V, size=20).astype(np.int32))),
                                                         float(a)) for a in rng.normal(size=16)])
            t = C.c_int64()
            _lib.check(L.fm_train_micro_batch(h, arr, 16, 16, C.byref(t)))
            g = np.empty(V * D)
            _lib.check(L.fm_agent_read_grad(h, g.ctypes.data))
            assert np.all(np.isfinite(g)), (V, D)
        finally:
            L.fm_agent_destroy(h)


@pytest.mark.parametrize("V,D,resp", [(2048, 4096, 24), (1000, 256, 200)])
def test_batched_reduction_equals_per_micro_batch(ctx, V, D, resp):
    """The step's K-GEMM2 is queued and runs once for all of its micro-batches
    (one TMEM accumulator with per-unit snapshots for short segments — the
    first shape, ~9 positions per 256-feature block — or double-buffered
    per-unit drains — the second).  Against the same step with every
    micro-batch's reduction forced by fm_agent_sync: the gradient, every
    micro-batch report (grad norm and loss) and the update agree to fp32
    summation order."""
    L = _lib.lib()
    rng = np.random.default_rng(V + D)
    W0 = np.ascontiguousarray(rng.normal(size=(V, D)) * 0.5)
    batches = [[(rng.integers(0, V, size=6).astype(np.int32), rng.integers(0, V, size=resp).astype(np.int32))
                for _ in range(4)] for _ in range(4)]
    advs = [rng.normal(size=4) for _ in range(4)]

    def run(sync_each):
        h = C.c_void_p()
        _lib.check(L.fm_agent_create(ctx.handle, b"q", V, D, _lib.PRECISION_BF16_TC, C.byref(h)))
        try:
            _lib.check(L.fm_agent_set_weights(h, W0.ctypes.data))
            tickets = []
            for k in range(4):
                arr = (_lib.fm_sample * 4)(*[_lib.fm_sample(ctx.put(orc.encode(p)), ctx.put(orc.encode(r)), float(a))
                                             for (p, r), a in zip(batches[k], advs[k])])
                t = C.c_int64()
                _lib.check(L.fm_train_micro_batch(h, arr, 4, 16, C.byref(t)))
                tickets.append(t.value)
                if sync_each:
                    _lib.check(L.fm_agent_sync(h))
            g = np.empty(V * D)
            _lib.check(L.fm_agent_read_grad(h, g.ctypes.data))
            reps = []
            for t in tickets:
                rep = _lib.fm_report()
                assert L.fm_agent_poll_report(h, t, C.byref(rep)) in (0, 1)
                _lib.check(L.fm_agent_sync(h))
                assert L.fm_agent_poll_report(h, t, C.byref(rep)) == 1
                reps.append((rep.grad_norm, rep.loss))
            gn = C.c_double()
            _lib.check(L.fm_apply_update(h, 16, 1e-3, 0.9, 0.999, 1e-8, C.byref(gn), None))
            W = np.empty(V * D)
            _lib.check(L.fm_agent_read_weights(h, W.ctypes.data))
            return g, np.array(reps), gn.value, W
        finally:
            L.fm_agent_destroy(h)

    g1, r1, n1, W1 = run(True)
    g4, r4, n4, W4 = run(False)
    assert np.all(np.isfinite(g4)) and np.any(g4 != 0)
    assert rel_fro(g4, g1) < 1e-5
    np.testing.assert_allclose(r4, r1, rtol=1e-4)
    assert abs(n4 - n1) <= 1e-5 * n1
    assert rel_fro(W4 - W0.reshape(-1), W1 - W0.reshape(-1)) < 1e-3


@pytest.mark.parametrize("tier", [_lib.TIER_HOST, _lib.TIER_DEVICE])
def test_queued_reduction_survives_swap(ctx, tier):
    """Two micro-batches queued (their K-GEMM2 not yet run), the agent
    suspended and re-activated, two more trained, then the update: the
    suspend runs the queued reduction first (check_active), the partial dW
    travels with the parked state, and the result equals the uninterrupted
    step's (same queue boundaries: 2 + 2 vs 4 units, fp32 summation order)."""
    L = _lib.lib()
    V, D = 1024, 512
    rng = np.random.default_rng(23)
    W0 = np.ascontiguousarray(rng.normal(size=(V, D)) * 0.5)
    batches = [[(rng.integers(0, V, size=6).astype(np.int32), rng.integers(0, V, size=40).astype(np.int32))
                for _ in range(4)] for _ in range(4)]
    advs = [rng.normal(size=4) for _ in range(4)]

    def run(swap):
        h = C.c_void_p()
        _lib.check(L.fm_agent_create(ctx.handle, b"s", V, D, _lib.PRECISION_BF16_TC, C.byref(h)))
        try:
            _lib.check(L.fm_agent_set_weights(h, W0.ctypes.data))
            tickets = []
            for k in range(4):
                if swap and k == 2:
                    _lib.check(L.fm_agent_suspend(h, tier, -1))
                    _lib.check(L.fm_agent_activate(h, ctx.handle))
                arr = (_lib.fm_sample * 4)(*[_lib.fm_sample(ctx.put(orc.encode(p)), ctx.put(orc.encode(r)), float(a))
                                             for (p, r), a in zip(batches[k], advs[k])])
                t = C.c_int64()
                _lib.check(L.fm_train_micro_batch(h, arr, 4, 16, C.byref(t)))
                tickets.append(t.value)
            gn = C.c_double()
            _lib.check(L.fm_apply_update(h, 16, 1e-3, 0.9, 0.999, 1e-8, C.byref(gn), None))
            norms = []
            for t in tickets:
                rep = _lib.fm_report()
                assert L.fm_agent_poll_report(h, t, C.byref(rep)) in (0, 1)
                _lib.check(L.fm_agent_sync(h))
                assert L.fm_agent_poll_report(h, t, C.byref(rep)) == 1
                norms.append(rep.grad_norm)
            W = np.empty(V * D)
            _lib.check(L.fm_agent_read_weights(h, W.ctypes.data))
            return np.array(norms), gn.value, W
        finally:
            L.fm_agent_destroy(h)

    n0, u0, W0r = run(False)
    n1, u1, W1r = run(True)
    assert np.all(np.isfinite(n1)) and np.all(n1 > 0)
    np.testing.assert_allclose(n1, n0, rtol=1e-4)
    assert abs(u1 - u0) <= 1e-5 * u0
    assert rel_fro(W1r - W0.reshape(-1), W0r - W0.reshape(-1)) < 1e-3
