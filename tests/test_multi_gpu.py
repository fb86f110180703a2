"""Multi-GPU tests: run tests/dp_check.py under torchrun when the box has
>= 2 GPUs (skipped on single-GPU boxes)."""
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("mode,norms,port", [("allreduce", "", 29511), ("gang", "", 29512),
                                           ("allreduce", "norms", 29514), ("gang", "norms", 29515),
                                           ("vocab", "", 29516)])
def test_dp_gang_parity(mode, norms, port, n=2):
    """DP gang of 2 vs the reference golden run; with "norms" the exact
    per-micro-batch grad norms (fm_agent_set_dp_norms) against the reference's;
    "vocab" is the vocabulary-parallel gang (exact norms by construction)."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
                        "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "tests" / "dp_check.py"),
                        mode] + ([norms] if norms else []), capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout


@pytest.mark.skipif(_ngpu() < 4, reason="needs >= 4 GPUs")
@pytest.mark.parametrize("mode,port", [("gang", 29517), ("vocab", 29518)])
def test_dp_gang_parity_4(mode, port):
    """The same checks with a gang of 4 (V=1000: one 256-row tile per rank)."""
    test_dp_gang_parity(mode, "", port, n=4)


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("how,port", [("migrate", 29513), ("share", 29521)])
def test_cross_process_migration(how, port):
    """migrate: export parks the agent, the importer finishes the step; share:
    fm_agent_share_export keeps it active on the exporter as well."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", f"--master-port={port}", str(ROOT / "tests" / "migrate_check.py"),
                        how], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout, r.stdout[-3000:]


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("tier", ["peer", "device"])
@pytest.mark.parametrize("back_on", [0, 1])
def test_peer_tier_swap_identity(back_on, tier):
    """FM_TIER_PEER (training.hpp:321-350 / 259-317 with the state parked in a
    peer GPU's HBM over NVLink, cudaMemcpyPeerAsync on the copy streams): an
    agent with a mid-step gradient suspended from GPU 0 into GPU 1's HBM and
    re-activated on GPU 0 or GPU 1 has a bit-identical state checksum, and the
    next micro-batch gives the same gradient as an agent that never moved."""
    import ctypes as C

    import numpy as np

    from oracle import oracle as orc
    from paper_2602_09578_b200 import _lib
    from paper_2602_09578_b200.engine import Context
    L = _lib.lib()
    V, D = 2048, 256
    rng = np.random.default_rng(3)
    W0 = np.ascontiguousarray(rng.normal(size=(V, D)) * 0.5)
    batches = [[(rng.integers(0, V, size=6).astype(np.int32), rng.integers(0, V, size=40).astype(np.int32))
                for _ in range(16)] for _ in range(2)]
    advs = [rng.normal(size=16) for _ in range(2)]
    ctxs = [Context(0), Context(1)]

    def train(h, ctx, k):
        arr = (_lib.fm_sample * 16)(*[_lib.fm_sample(ctx.put(orc.encode(p)), ctx.put(orc.encode(r)), a)
                                      for (p, r), a in zip(batches[k], advs[k])])
        t = C.c_int64()
        _lib.check(L.fm_train_micro_batch(h, arr, 16, 64, C.byref(t)))

    def checksum(h):
        cs = C.c_uint64()
        _lib.check(L.fm_agent_state_checksum(h, C.byref(cs)))
        return cs.value

    hs = []
    try:
        for name in (b"moved", b"stayed"):
            h = C.c_void_p()
            _lib.check(L.fm_agent_create(ctxs[0].handle, name, V, D, _lib.PRECISION_BF16_TC, C.byref(h)))
            _lib.check(L.fm_agent_set_weights(h, W0.ctypes.data))
            hs.append(h)
            train(h, ctxs[0], 0)
        moved, stayed = hs
        before = checksum(moved)
        assert before == checksum(stayed)
        if tier == "peer":
            _lib.check(L.fm_agent_suspend(moved, _lib.TIER_PEER, 1))
        else:  # parked in GPU 0's HBM; activation on GPU 1 pulls it over NVLink
            _lib.check(L.fm_agent_suspend(moved, _lib.TIER_DEVICE, -1))
            assert L.fm_agent_is_active(moved) == 0
        _lib.check(L.fm_agent_activate(moved, ctxs[back_on].handle))
        assert checksum(moved) == before
        train(moved, ctxs[back_on], 1)
        train(stayed, ctxs[0], 1)
        g_m = np.empty(V * D)
        g_s = np.empty(V * D)
        _lib.check(L.fm_agent_read_grad(moved, g_m.ctypes.data))
        _lib.check(L.fm_agent_read_grad(stayed, g_s.ctypes.data))
        np.testing.assert_array_equal(g_m, g_s)
    finally:
        for h in hs:
            L.fm_agent_destroy(h)
        for c in ctxs:
            c.close()


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_weight_broadcast():
    """fm_weights_broadcast: every dtype arrives byte-identical with the root's
    version on the other rank (tests/bcast_check.py)."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", "--master-port=29519", str(ROOT / "tests" / "bcast_check.py")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "weight broadcast OK" in r.stdout, r.stdout[-3000:]


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_gang_dissolve():
    """fm_gang_gather_state + fm_gang_detach (tests/gang_detach_check.py): the
    lead rank ends up with the gang's whole state, a whole bf16 shadow, and the
    gradients of a fresh one-GPU agent."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", "--master-port=29520", str(ROOT / "tests" / "gang_detach_check.py")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "-> OK" in r.stdout, r.stdout[-3000:]


@pytest.mark.skipif(_ngpu() < 2, reason="needs >= 2 GPUs")
def test_gang_from_row_range_import():
    """fm_agent_migrate_import_rows (tests/rows_import_check.py): a vocabulary
    gang formed from a rank's own-rows import trains bit-identically to one
    formed from a whole import; the partial agent is refused elsewhere."""
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr=127.0.0.1", "--master-port=29522", str(ROOT / "tests" / "rows_import_check.py")],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "-> OK" in r.stdout, r.stdout[-3000:]
