"""Weight sync by NCCL broadcast (run under torchrun, >= 2 GPUs):
`fm_weights_broadcast` (the rollout-sync path; publish_weights
training.hpp:459-467 + the rollout engines' Get, rollout.hpp:510-541).

Rank 0 publishes one agent's weights in every dtype (0 f64 payload, 1 f32,
2 bf16, 3 f64 transposed [D][V]); every other rank allocates an empty buffer of
the same shape and dtype and receives it in one broadcast.  Each rank checks
its received bytes (read back with `fm_weights_get`) and version against the
root's: byte-identical, version stamped."""
import ctypes as C
import hashlib
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import torch.distributed as dist  # noqa: E402

from paper_2602_09578_b200 import _lib  # noqa: E402
from paper_2602_09578_b200.engine import Context  # noqa: E402


def main():
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
    V, D = 1000, 136
    W0 = np.random.default_rng(5).normal(size=(V, D))
    h = C.c_void_p()
    ok = True
    if rank == 0:
        _lib.check(L.fm_agent_create(ctx.handle, b"src", V, D, _lib.PRECISION_BF16_TC, C.byref(h)))
        _lib.check(L.fm_agent_set_weights(h, np.ascontiguousarray(W0).ctypes.data))
    for dtype, esz in ((0, 8), (1, 4), (2, 2), (3, 8)):
        w = C.c_void_p()
        if rank == 0:
            _lib.check(L.fm_publish_weights(h, dtype, C.byref(w)))
        else:
            _lib.check(L.fm_weights_alloc(ctx.handle, V, D, dtype, C.byref(w)))
        _lib.check(L.fm_weights_broadcast(w, comm, 0))
        host = np.empty(V * D * esz, np.uint8)
        _lib.check(L.fm_weights_get(w, host.ctypes.data, -1))
        ver = C.c_int64()
        _lib.check(L.fm_weights_info(w, C.byref(ver), None, None, None, None, None))
        digests = [None] * world
        dist.all_gather_object(digests, (hashlib.sha1(host.tobytes()).hexdigest(), ver.value))
        same = len(set(digests)) == 1
        if dtype == 0:  # the reference payload: W's f64 bytes
            same = same and host.tobytes() == np.ascontiguousarray(W0).tobytes()
        elif dtype == 3:
            same = same and host.tobytes() == np.ascontiguousarray(W0.T).tobytes()
        if not same:
            print(f"rank {rank}: dtype {dtype} broadcast differs: {digests}", flush=True)
        ok = ok and same
        _lib.check(L.fm_weights_destroy(w))
    if rank == 0:
        L.fm_agent_destroy(h)
    L.fm_comm_destroy(comm)
    ctx.close()
    import torch
    okt = torch.tensor([1 if ok else 0])
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    if rank == 0:
        print("weight broadcast " + ("OK" if okt.item() == 1 else "FAIL"), flush=True)
    dist.destroy_process_group()
    sys.exit(0 if okt.item() == 1 else 1)


if __name__ == "__main__":
    main()
