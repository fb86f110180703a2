"""Cross-process agent migration over NVLink (run under torchrun, 2 GPUs).

Rank 0 trains two micro-batches of a step (a pending gradient, Adam moments of
an earlier update), exports the agent (fm_agent_migrate_export: park in its HBM
+ CUDA IPC handles); rank 1 imports it into a fresh agent on its own GPU
(copy-engine peer copies) and finishes the step (two more micro-batches +
update).  Checks:
  * the imported state's checksum equals the exported one (identity swap);
  * version / Adam step / accumulated samples travel with it;
  * the migrated run's final W, m, v equal an unmigrated run of the same
    micro-batches on rank 0's GPU bit for bit (same kernels, same inputs).
With argument "share" rank 0 exports with fm_agent_share_export instead (the
agent stays active there, as when a DP gang forms around it — bench.py C4) and
finishes the step itself as well: both copies must end bit-identical.
"""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch  # noqa: E402,F401
import torch.distributed as dist  # noqa: E402

import workload_helpers as wh  # noqa: E402
from paper_2602_09578_b200 import _lib  # noqa: E402
from paper_2602_09578_b200.engine import Context  # noqa: E402

L = _lib.lib()
V, D, G, MB = 1000, 64, 64, 16


def batches():
    rng = np.random.default_rng(21)
    return [[(rng.integers(0, V, 6).astype(np.int32), rng.integers(0, V, 60).astype(np.int32), float(a))
             for a in rng.normal(size=MB)] for _ in range(2 * G // MB)]


def train(ctx, h, bts):
    for bt in bts:
        arr = (_lib.fm_sample * MB)(*[_lib.fm_sample(ctx.put(wh.enc(p)), ctx.put(wh.enc(r)), a) for p, r, a in bt])
        t = C.c_int64()
        _lib.check(L.fm_train_micro_batch(h, arr, MB, G, C.byref(t)))
        if _lib.lib().fm_agent_samples_accumulated(h) == G:
            _lib.check(L.fm_apply_update(h, G, 1e-3, 0.9, 0.999, 1e-8, None, None))


def state(h):
    P = V * D
    w, m, v = np.empty(P), np.empty(P, np.float32), np.empty(P, np.float32)
    step = C.c_int64()
    _lib.check(L.fm_agent_read_weights(h, w.ctypes.data))
    _lib.check(L.fm_agent_read_moments(h, m.ctypes.data, v.ctypes.data, C.byref(step)))
    return w, m, v, step.value


def checksum(h):
    out = C.c_uint64()
    _lib.check(L.fm_agent_state_checksum(h, C.byref(out)))
    return out.value


def main():
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    share = len(sys.argv) > 1 and sys.argv[1] == "share"
    local = int(os.environ.get("LOCAL_RANK", rank))
    ctx = Context(local)
    bts = batches()  # step 1 = bts[0:4], step 2 = bts[4:8]
    W0 = np.ascontiguousarray(np.random.default_rng(3).normal(size=(V, D)) * 0.5)
    h = C.c_void_p()
    _lib.check(L.fm_agent_create(ctx.handle, b"mover", V, D, _lib.PRECISION_BF16_TC, C.byref(h)))
    ok = True
    if rank == 0:
        _lib.check(L.fm_agent_set_weights(h, W0.ctypes.data))
        train(ctx, h, bts[:6])  # one full step + half of the second: pending gradient
        before = (checksum(h), L.fm_agent_version(h), L.fm_agent_samples_accumulated(h))
        n = C.c_uint64()
        export = L.fm_agent_share_export if share else L.fm_agent_migrate_export
        _lib.check(export(h, None, 0, C.byref(n)))
        blob = (C.c_uint8 * n.value)()
        _lib.check(export(h, blob, n.value, C.byref(n)))
        dist.broadcast_object_list([bytes(blob), before], src=0)
        dist.barrier()  # rank 1 imported: the parked copy may go
        kept = None
        if share:  # still active here: finish the step on this GPU too
            train(ctx, h, bts[6:])
            kept = state(h)
        _lib.check(L.fm_agent_destroy(h))
        # the unmigrated reference run on this GPU
        h2 = C.c_void_p()
        _lib.check(L.fm_agent_create(ctx.handle, b"stay", V, D, _lib.PRECISION_BF16_TC, C.byref(h2)))
        _lib.check(L.fm_agent_set_weights(h2, W0.ctypes.data))
        train(ctx, h2, bts)
        ref = state(h2)
        got = [None]
        dist.broadcast_object_list(got, src=1)
        w, m, v, step = got[0]
        for name, a, b in (("W", w, ref[0]), ("m", m, ref[1]), ("v", v, ref[2])):
            if not np.array_equal(a, b):
                print(f"FAIL {name}: migrated run differs ({np.abs(a - b).max()})")
                ok = False
        if step != ref[3]:
            print(f"FAIL adam step {step} vs {ref[3]}")
            ok = False
        if kept is not None:
            for name, a, b in (("W", kept[0], ref[0]), ("m", kept[1], ref[1]), ("v", kept[2], ref[2])):
                if not np.array_equal(a, b):
                    print(f"FAIL {name}: the sharing rank's own run differs")
                    ok = False
        _lib.check(L.fm_agent_destroy(h2))
    else:
        msg = [None, None]
        dist.broadcast_object_list(msg, src=0)
        blob, before = msg
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        _lib.check(L.fm_agent_migrate_import(h, ctx.handle, buf, len(blob)))
        dist.barrier()
        after = (checksum(h), L.fm_agent_version(h), L.fm_agent_samples_accumulated(h))
        if after != before:
            print(f"FAIL imported state {after} vs exported {before}")
            ok = False
        train(ctx, h, bts[6:])
        dist.broadcast_object_list([state(h)], src=1)
        _lib.check(L.fm_agent_destroy(h))
    oks = [None] * dist.get_world_size()
    dist.all_gather_object(oks, ok)
    ctx.close()
    if rank == 0:
        print("OK" if all(oks) else "FAILED")
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
