"""Multi-GPU data-parallel parity (run under torchrun, >= 2 GPUs).

Every rank of one gang trains its token-balanced shard of each polled
micro-batch of the V=256/D=64 golden fixture, the gang all-reduces dW over
NCCL, and rank 0 checks the reduced gradient and the post-update weights
against the compiled-reference golden run (same tolerances as the 1-GPU
tensor-core path)."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import torch.distributed as dist  # noqa: E402

from paper_2602_09578_b200 import _lib  # noqa: E402
from paper_2602_09578_b200.engine import Context  # noqa: E402
from fixture_runner import payload  # noqa: E402
from test_gpu_path import _oracle_grad_step0, rel_fro  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    L = _lib.lib()
    f = np.load(ROOT / "tests" / "golden" / "mid_agent0.npz")
    V, D, G, mb, U = (int(f[k]) for k in ("V", "D", "G", "mb", "n_updates"))
    ctx = Context(local)
    uid = [None]
    if rank == 0:
        b = (C.c_uint8 * 128)()
        _lib.check(L.fm_comm_unique_id(b))
        uid = [bytes(b)]
    dist.broadcast_object_list(uid, src=0)
    comm = C.c_void_p()
    _lib.check(L.fm_comm_create(ctx.handle, (C.c_uint8 * 128).from_buffer_copy(uid[0]), world, rank, C.byref(comm)))
    h = C.c_void_p()
    _lib.check(L.fm_agent_create(ctx.handle, b"agent0", V, D, _lib.PRECISION_BF16_TC, C.byref(h)))
    _lib.check(L.fm_agent_set_weights(h, np.ascontiguousarray(f["W0"]).ctypes.data))
    _lib.check(L.fm_agent_set_shard(h, rank, world))
    po = f["poll_order"]
    grads = []
    for u in range(U):
        for b in range(G // mb):
            idx = po[u * G + b * mb: u * G + (b + 1) * mb]
            arr = (_lib.fm_sample * mb)(*[_lib.fm_sample(ctx.put(payload(f, int(f["prompt_off"][i]))),
                                                         ctx.put(payload(f, int(f["resp_off"][i]))),
                                                         float(f["adv"][i])) for i in idx])
            t = C.c_int64()
            _lib.check(L.fm_train_micro_batch(h, arr, mb, G, C.byref(t)))
        _lib.check(L.fm_agent_allreduce_grad(h, comm))
        g = np.empty(V * D)
        _lib.check(L.fm_agent_read_grad(h, g.ctypes.data))
        grads.append(g.reshape(V, D))
        _lib.check(L.fm_apply_update(h, G, 1e-6, 0.9, 0.999, 1e-8, None, None))
    W = np.empty(V * D)
    _lib.check(L.fm_agent_read_weights(h, W.ctypes.data))
    ok = True
    if rank == 0:
        g_ref = _oracle_grad_step0(f)
        e_g = rel_fro(grads[0], g_ref)
        dW, dW_ref = W.reshape(V, D) - f["W0"], f["W"] - f["W0"]
        e_w = rel_fro(dW, dW_ref)
        ok = e_g <= 2e-2 and e_w <= 5e-2
        print(f"DP world={world}: grad rel {e_g:.3e}, dW rel {e_w:.3e} -> {'OK' if ok else 'FAIL'}", flush=True)
    # all ranks must hold identical weights after the replicated update
    Wt = __import__("torch").tensor(W)
    ref = Wt.clone()
    dist.broadcast(ref, src=0)
    same = bool((Wt == ref).all())
    if not same:
        print(f"rank {rank}: weights diverged from rank 0", flush=True)
    L.fm_agent_destroy(h)
    L.fm_comm_destroy(comm)
    ctx.close()
    dist.destroy_process_group()
    sys.exit(0 if (ok and same) else 1)


if __name__ == "__main__":
    main()
