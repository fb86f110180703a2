"""Exercises the on-device experience table kernels at C2-like sizes for ncu
(tools/profile_round_v4.sh): a 256-record table (one-block poll), a 4,096-record
table (chunk candidates + rank + finish), and a release of 64 groups x 16
survivors with 1,024-token responses (K-release)."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_09578_b200.engine import Context, DeviceExperienceStore, SampleId, TableSchema  # noqa: E402


def main():
    ctx = Context(0)
    rng = np.random.default_rng(0)
    for nrec in (256, 4096):
        st = DeviceExperienceStore(ctx, capacity=nrec)
        st.create_table(TableSchema("a", [("advantage", "Float")]))
        ids = [SampleId(f"q{i // 16:05d}", 0, i % 16) for i in rng.permutation(nrec)]
        sl = st.insert_many("a", 0, ids)
        st.set_cells("a", "advantage", sl, np.zeros(nrec))
        while st.poll_micro_batch("a", 0, 16, columns=None) is not None:
            pass
        st.close()
    ngrp, k, L = 64, 16, 1024
    st = DeviceExperienceStore(ctx, capacity=ngrp * k)
    st.create_table(TableSchema("a", [("response", "List"), ("reward", "Float"), ("advantage", "Float")]))
    sl = st.insert_many("a", 0, [SampleId(f"q{i // k:05d}", 0, i % k) for i in range(ngrp * k)])
    for s in sl:
        t = rng.integers(0, 8, size=L).astype(np.uint64)
        st.set_payload_slot("a", "response", int(s), np.uint64(L).tobytes() + t.tobytes())
    st.release_groups([[(("a", int(sl[g * k + j])), [("a", int(sl[g * k + j]))]) for j in range(k)]
                       for g in range(ngrp)], read_back=True)
    st.close()
    ctx.close()
    print("ok")


if __name__ == "__main__":
    main()
