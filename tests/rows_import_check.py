"""Forming a vocabulary gang from a row-range import (run under torchrun, 2 GPUs):
`fm_agent_migrate_import_rows` (bench.py C4 re-placement: a rank joining a
vocabulary-parallel gang pulls only its own rows of W / m / v over NVLink).

Rank 0 trains two identical agents one solo step (so m / v are non-zero) and
share-exports both.  Rank 1 imports the first with only its vocabulary rows and
the second whole.  Checks:
  * the row-range agent refuses use outside its gang (ConfigError), and a range
    that is not the rank's is refused at attach;
  * gang 1 (rank 0 + the row-range import) and gang 2 (rank 0 + the whole
    import) train the same next step to bit-identical owner-assembled weights
    and PolicyState bytes."""
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
from gang_detach_check import serialize  # noqa: E402

ERR_CONFIG = _lib.ERROR_NAMES.index("ConfigError")  # FM_ERR_CONFIG_ERROR (cabi.h)


def main():
    import workload_helpers as wh
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    assert world == 2
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
    tiles = (V + 255) // 256
    lo = [min(V, (tiles * o // world) * 256) for o in range(world + 1)]
    rng = np.random.default_rng(29)
    W0 = np.ascontiguousarray(rng.normal(size=(V, D)) * 0.5)
    steps = [[[(rng.integers(0, V, 5).astype(np.int32), rng.integers(0, V, 40).astype(np.int32), float(a))
               for a in rng.normal(size=mb)] for _ in range(G // mb)] for _ in range(2)]

    def train_step(h, step):
        for bt in step:
            arr = (_lib.fm_sample * mb)(*[_lib.fm_sample(ctx.put(wh.enc(p)), ctx.put(wh.enc(r)), a)
                                          for p, r, a in bt])
            t = C.c_int64()
            _lib.check(L.fm_train_micro_batch(h, arr, mb, G, C.byref(t)))
        _lib.check(L.fm_apply_update(h, G, 1e-3, 0.9, 0.999, 1e-8, None, None))
        _lib.check(L.fm_agent_sync(h))

    def new_agent(name):
        h = C.c_void_p()
        _lib.check(L.fm_agent_create(ctx.handle, name, V, D, _lib.PRECISION_BF16_TC, C.byref(h)))
        return h

    ok = True
    blobs = [None, None]
    src = []
    if rank == 0:
        for k in range(2):
            h = new_agent(f"src{k}".encode())
            _lib.check(L.fm_agent_set_weights(h, W0.ctypes.data))
            train_step(h, steps[0])
            n = C.c_uint64()
            _lib.check(L.fm_agent_share_export(h, None, 0, C.byref(n)))
            buf = (C.c_uint8 * n.value)()
            _lib.check(L.fm_agent_share_export(h, buf, n.value, C.byref(n)))
            blobs[k] = bytes(buf)
            src.append(h)
        ok = serialize(L, src[0], G).tobytes() == serialize(L, src[1], G).tobytes()
    dist.broadcast_object_list(blobs, src=0)
    dst = []
    if rank == 1:
        part, full, wrong = new_agent(b"part"), new_agent(b"full"), new_agent(b"wrong")
        for h, blob, rows in ((part, blobs[0], (lo[1], lo[2])), (full, blobs[1], None), (wrong, blobs[0], (0, 256))):
            buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
            if rows is None:
                _lib.check(L.fm_agent_migrate_import(h, ctx.handle, buf, len(blob)))
            else:
                _lib.check(L.fm_agent_migrate_import_rows(h, ctx.handle, buf, len(blob), rows[0], rows[1]))
        Wtmp = np.empty(V * D)
        refused = L.fm_agent_read_weights(part, Wtmp.ctypes.data) == ERR_CONFIG
        n = C.c_uint64()
        blob = (C.c_uint8 * 4096)()
        bad_range = L.fm_gang_attach_mode(wrong, comm, 1, blob, 4096, C.byref(n)) == ERR_CONFIG
        L.fm_agent_destroy(wrong)
        if not (refused and bad_range):
            print(f"row-range agent: refused outside its gang {refused}, wrong range refused {bad_range}", flush=True)
        ok = refused and bad_range
        dst = [part, full]
    dist.barrier()  # every importer returned: the sources may run again

    results = []
    for k in range(2):
        h = src[k] if rank == 0 else dst[k]
        _attach(L, h, comm, world, 1)
        train_step(h, steps[1])
        dist.barrier()  # every owner's rows are final
        if rank == 0:
            W = np.empty(V * D)
            _lib.check(L.fm_agent_read_weights(h, W.ctypes.data))
            results.append((W, serialize(L, h, G).tobytes()))
        dist.barrier()
        _lib.check(L.fm_gang_detach(h))
        L.fm_agent_destroy(h)
    if rank == 0:
        same = bool(np.array_equal(results[0][0], results[1][0])) and results[0][1] == results[1][1]
        ok = ok and same
        print(f"vocabulary gang from a row-range import: weights and state "
              f"{'bit-identical' if same else 'DIFFER'} to the whole-import gang -> {'OK' if ok else 'FAIL'}",
              flush=True)
    L.fm_comm_destroy(comm)
    ctx.close()
    okt = torch.tensor([1 if ok else 0])
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    sys.exit(0 if okt.item() == 1 else 1)


if __name__ == "__main__":
    main()
