"""Replays a golden store script (tests/golden/store_script_*.txt) on the
on-device experience table, producing the reference driver's result lines
(oracle/ref_driver.cpp ref_store_script) so the two compare as text."""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle.store_oracle import StoreError, hexf, parse_release, replay  # noqa: E402
from paper_2602_09578_b200 import _lib  # noqa: E402
from paper_2602_09578_b200.engine import DeviceExperienceStore, SampleId, TableSchema  # noqa: E402

SCHEMA = [("prompt", "List"), ("response", "List"), ("logprobs", "Tensor"), ("reward", "Float"),
          ("advantage", "Float")]


def codec(tokens) -> bytes:  # encode_tokens (codec.hpp:15-22)
    t = np.asarray(tokens, np.int64).astype(np.uint64)
    return np.uint64(len(t)).tobytes() + t.tobytes()


class DeviceAdapter:
    def __init__(self, ctx, capacity=1024):
        self.st = DeviceExperienceStore(ctx, capacity)
        self.st.create_table(TableSchema("agent", SCHEMA))
        self.A = "agent"

    def close(self):
        self.st.close()

    def op(self, op, a):
        try:
            return self._op(op, a)
        except _lib.FlexMarlError as e:
            raise StoreError(e.code)

    def _op(self, op, a):
        st, A = self.st, self.A
        sid = lambda i: SampleId(a[i], int(a[i + 1]), int(a[i + 2]))  # noqa: E731
        if op == "insert":
            st.insert(A, int(a[0]), sid(1))
            return "ok"
        if op == "setf":
            st.set_cell(A, sid(1), int(a[0]), a[4], float.fromhex(a[5]))
            return "ok"
        if op == "setp":
            st.set_cell_payload(A, sid(1), int(a[0]), a[4], codec([int(x) for x in a[6:6 + int(a[5])]]))
            return "ok"
        if op == "poll":
            b = st.poll_micro_batch(A, int(a[0]), int(a[1]))
            if b is None:
                return "none"
            adv = st.read_cells(A, "advantage", [s.handle for s in b.samples])
            return " ".join(f"{s.sample_id.render()}@{s.policy_version}:{hexf(float(x))}"
                            for s, x in zip(b.samples, adv))
        if op == "complete":
            k = int(a[0])
            slots = [st.find(A, SampleId(a[2 + 4 * i], int(a[3 + 4 * i]), int(a[4 + 4 * i])), int(a[1 + 4 * i]))
                     for i in range(k)]
            hs = np.ascontiguousarray(slots or [0], np.int64)
            _lib.check(_lib.lib().fm_dtable_complete(st.table(A), hs.ctypes.data, k))
            return "ok"
        if op == "purge_stale":
            return str(st.purge_stale(A, int(a[0])))
        if op == "purge_inputs":
            return str(st.purge_inputs(A, a[1:1 + int(a[0])]))
        if op == "drop":
            return "1" if st.drop_record(A, sid(1), int(a[0])) else "0"
        if op == "ready":
            return str(st.ready_count(A, int(a[0])))
        if op == "count":
            return str(st.record_count(A))
        if op == "release":
            eps, pat, surv = parse_release(a)
            grp = []
            for (gid, t, j, v), recs in surv:
                grp.append(((A, st.find(A, SampleId(gid, t, j), v)),
                            [(A, st.find(A, SampleId(x, tt, jj), vv)) for (x, tt, jj, vv) in recs]))
            rew, adv = st.release_groups([grp], pattern=pat, eps_adv=eps, read_back=True)
            return " ".join(f"{hexf(float(r))}/{hexf(float(d))}" for r, d in zip(rew, adv)) or "ok"
        return "bad-op"


def replay_device(ctx, script: str) -> str:
    ad = DeviceAdapter(ctx)
    try:
        return replay(script, ad)
    finally:
        ad.close()
