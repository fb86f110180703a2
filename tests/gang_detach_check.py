"""Dissolving a vocabulary-parallel gang (run under torchrun, >= 2 GPUs): the
C4 re-placement path (bench.py `transition`).

A gang of `world` ranks trains one global step of a V=1000 agent (each rank
keeps only its own vocabulary columns of W / m / v / W16^T current).  Rank 0
then pulls the peers' rows (`fm_gang_gather_state`), every rank detaches
(`fm_gang_detach`), and rank 0 must hold the whole training state:
  * its serialized PolicyState equals the one the gang assembled from the
    owners before the dissolve (byte-identical: W, m, v, version);
  * its rebuilt bf16 shadow is bf16(W) (the bf16 publish untransposes it);
  * the next micro-batch's gradient equals that of a fresh one-GPU agent
    loaded with the same weights (bit-identical: same shadow, same kernels)."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2602_09578_b200 import _lib  # noqa: E402
from paper_2602_09578_b200.engine import Context  # noqa: E402
from dp_check import _attach  # noqa: E402


def serialize(L, h, G):
    n = C.c_uint64()
    _lib.check(L.fm_agent_serialize(h, G, None, 0, C.byref(n)))
    blob = np.empty(n.value, np.uint8)
    _lib.check(L.fm_agent_serialize(h, G, blob.ctypes.data, n.value, C.byref(n)))
    return blob


def main():
    import workload_helpers as wh
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    L = _lib.lib()
    ctx = Context(int(os.environ.get("LOCAL_RANK", rank)))
    uid = [None]
    if rank == 0:
        b = (C.c_uint8 * 128)()
        _lib.check(L.fm_comm_unique_id(b))
        uid = [bytes(b)]
    dist.broadcast_object_list(uid, src=0)
    comm = C.c_void_p()
    _lib.check(L.fm_comm_create(ctx.handle, (C.c_uint8 * 128).from_buffer_copy(uid[0]), world, rank, C.byref(comm)))

    V, D, G, mb = 1000, 72, 32, 16
    rng = np.random.default_rng(17)
    W0 = rng.normal(size=(V, D)) * 0.5
    batches = [[(rng.integers(0, V, 5).astype(np.int32), rng.integers(0, V, 40).astype(np.int32), float(a))
                for a in rng.normal(size=mb)] for _ in range(G // mb + 1)]

    def train(h, bt):
        arr = (_lib.fm_sample * mb)(*[_lib.fm_sample(ctx.put(wh.enc(p)), ctx.put(wh.enc(r)), a) for p, r, a in bt])
        t = C.c_int64()
        _lib.check(L.fm_train_micro_batch(h, arr, mb, G, C.byref(t)))

    h = C.c_void_p()
    _lib.check(L.fm_agent_create(ctx.handle, b"gang", V, D, _lib.PRECISION_BF16_TC, C.byref(h)))
    _lib.check(L.fm_agent_set_weights(h, np.ascontiguousarray(W0).ctypes.data))
    _attach(L, h, comm, world, 1)
    for bt in batches[:-1]:
        train(h, bt)
    _lib.check(L.fm_apply_update(h, G, 1e-3, 0.9, 0.999, 1e-8, None, None))
    _lib.check(L.fm_agent_sync(h))
    dist.barrier()  # every owner's rows are final
    before = serialize(L, h, G)  # assembled from the owners' rows (every rank the same bytes)
    dist.barrier()
    if rank == 0:
        _lib.check(L.fm_gang_gather_state(h))
    dist.barrier()
    _lib.check(L.fm_gang_detach(h))
    ok = True
    if rank == 0:
        after = serialize(L, h, G)
        same_state = before.tobytes() == after.tobytes()
        W = np.empty(V * D)
        _lib.check(L.fm_agent_read_weights(h, W.ctypes.data))
        w = C.c_void_p()
        _lib.check(L.fm_publish_weights(h, 2, C.byref(w)))
        out = torch.empty(V * D, dtype=torch.bfloat16)
        _lib.check(L.fm_weights_get(w, out.data_ptr(), -1))
        _lib.check(L.fm_weights_destroy(w))
        same_shadow = bool((out.view(torch.int16) == torch.tensor(W).float().bfloat16().view(torch.int16)).all())
        # the next micro-batch, standalone, against a fresh agent with the same weights
        grads = []
        for name, hh in (("detached", h), ("fresh", None)):
            if hh is None:
                hh = C.c_void_p()
                _lib.check(L.fm_agent_create(ctx.handle, b"fresh", V, D, _lib.PRECISION_BF16_TC, C.byref(hh)))
                _lib.check(L.fm_agent_set_weights(hh, W.ctypes.data))
            train(hh, batches[-1])
            g = np.empty(V * D)
            _lib.check(L.fm_agent_read_grad(hh, g.ctypes.data))
            grads.append(g)
            if name == "fresh":
                L.fm_agent_destroy(hh)
        same_grad = bool(np.array_equal(grads[0], grads[1]))
        ok = same_state and same_shadow and same_grad
        print(f"gang of {world} dissolved onto rank 0: state {'same' if same_state else 'DIFFERS'}, "
              f"shadow {'bf16(W)' if same_shadow else 'WRONG'}, next gradient "
              f"{'bit-identical' if same_grad else 'DIFFERS'} -> {'OK' if ok else 'FAIL'}", flush=True)
    L.fm_agent_destroy(h)
    L.fm_comm_destroy(comm)
    ctx.close()
    okt = torch.tensor([1 if ok else 0])
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    sys.exit(0 if okt.item() == 1 else 1)


if __name__ == "__main__":
    main()
