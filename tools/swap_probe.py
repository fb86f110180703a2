"""Probe: cost of a device-tier state swap (suspend + activate) of a C2 agent,
alone and overlapped with another agent's micro-batch (bench-like timing)."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_09578_b200 import _lib, workload as wl  # noqa: E402
from paper_2602_09578_b200.engine import Context  # noqa: E402

L = _lib.lib()
cfg = wl.CONFIGS["C2"]
ctx = Context(0)
ctx.reserve(64 << 20, 16 * 1024, cfg.vocab, cfg.feat)
hs = []
for n in (b"a", b"b"):
    h = C.c_void_p()
    _lib.check(L.fm_agent_create(ctx.handle, n, cfg.vocab, cfg.feat, 0, C.byref(h)))
    hs.append(h)
samples = wl.step_samples(cfg, "agent0", 0, n=16)
arr = (_lib.fm_sample * 16)(*[_lib.fm_sample(ctx.put(s.prompt_payload), ctx.put(s.response_payload), 0.5)
                              for s in samples])
ms = C.c_double()
t = C.c_int64()


def timed(fn, reps=3):
    out = []
    for _ in range(reps):
        ctx.synchronize()
        _lib.check(L.fm_ctx_timer_start(ctx.handle))
        fn()
        _lib.check(L.fm_ctx_timer_stop(ctx.handle, C.byref(ms)))
        out.append(ms.value)
    return min(out)


for tier, name in ((1, "device"), (0, "host")):
    def swap():
        _lib.check(L.fm_agent_suspend(hs[1], tier, -1))
        _lib.check(L.fm_agent_activate(hs[1], ctx.handle))

    def mb():
        _lib.check(L.fm_train_micro_batch(hs[0], arr, 16, 64, C.byref(t)))

    def both():
        swap()
        mb()
    print(f"{name}: swap {timed(swap):.2f} ms, micro-batch {timed(mb):.2f} ms, overlapped {timed(both):.2f} ms",
          flush=True)
