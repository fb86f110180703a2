"""Small end-to-end run of every hot-path kernel for compute-sanitizer
(memcheck / racecheck / synccheck, one tool per invocation; logs under
profiles/): K-gather / K-pos / K-pslot / K-fmax / K-stats / K-lse / K-band /
K-GEMM2 (tcgen05, TMA reduce-add epilogue) / K-adam (transposed shadow) /
update-and-park + swap-in, on ragged shapes (V, D not multiples of 256, V not
a multiple of 8, short and empty prompts, one-token responses)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from oracle import oracle as orc  # noqa: E402
from paper_2602_09578_b200 import _lib  # noqa: E402
from paper_2602_09578_b200.engine import Context  # noqa: E402


def main():
    L = _lib.lib()
    ctx = Context(0)
    for V, D, n, resp in [(300, 72, 5, 7), (2100, 520, 16, 33), (4100, 96, 3, 1)]:
        rng = np.random.default_rng(V + D)
        h = C.c_void_p()
        _lib.check(L.fm_agent_create(ctx.handle, b"san", V, D, _lib.PRECISION_BF16_TC, C.byref(h)))
        W0 = np.ascontiguousarray(rng.normal(size=(V, D)) * 0.5)
        _lib.check(L.fm_agent_set_weights(h, W0.ctypes.data))
        for step in range(2):
            for mb in range(2):
                samples = [([int(x) for x in rng.integers(0, 3 * V, size=int(rng.integers(0, 6)))],
                            [int(x) for x in rng.integers(0, V, size=resp)]) for _ in range(n)]
                arr = (_lib.fm_sample * n)(*[_lib.fm_sample(ctx.put(orc.encode(p)), ctx.put(orc.encode(r)), a)
                                             for (p, r), a in zip(samples, rng.normal(size=n))])
                t = C.c_int64()
                _lib.check(L.fm_train_micro_batch(h, arr, n, 2 * n, C.byref(t)))
            if step == 0:
                _lib.check(L.fm_apply_update_park(h, 2 * n, 1e-3, 0.9, 0.999, 1e-8, None, None))
                _lib.check(L.fm_agent_activate(h, ctx.handle))
            else:
                _lib.check(L.fm_apply_update(h, 2 * n, 1e-3, 0.9, 0.999, 1e-8, None, None))
        _lib.check(L.fm_agent_sync(h))
        L.fm_agent_destroy(h)
    ctx.close()
    print("sanitize run OK")


if __name__ == "__main__":
    main()
