"""Drives a golden fixture through the B200 engine exactly as the reference
driver (oracle/ref_driver.cpp) drives the reference: insert in the fixture's
insertion order, set payload/advantage cells, poll micro-batches in canonical
order, train, complete, apply the global update."""
from __future__ import annotations

import numpy as np

from paper_2602_09578_b200 import _lib
from paper_2602_09578_b200.engine import (ExperienceStore, SampleId, TableSchema, TrainingEngine)

SCHEMA_COLS = [("prompt", "List"), ("response", "List"), ("advantage", "Float")]


def payload(f, off):
    buf = f["payloads"]
    n = int(np.frombuffer(buf[off:off + 8].tobytes(), "<u8")[0])
    return buf[off:off + 8 + 8 * n].tobytes()


def run_fixture(ctx, f, precision, hooks=None):
    """Returns dict(poll_order, mb_grad_norm, upd_grad_norm, W, m, v, grads[list per update])."""
    agent = str(f["agent"])
    V, D, G, mb, U = (int(f[k]) for k in ("V", "D", "G", "mb", "n_updates"))
    ctx.reset_arena()
    store = ExperienceStore(ctx)
    schema = TableSchema(agent, SCHEMA_COLS)
    store.create_table(schema)
    eng = TrainingEngine([ctx], global_batch=G, precision=precision)
    eng.add_agent(agent, V, D)
    eng.activate(agent)
    eng.run()
    key_to_idx = {(str(f["ids"][i]), int(f["turns"][i]), int(f["trajs"][i]), int(f["versions"][i])): i
                  for i in range(len(f["ids"]))}
    polled, mbn, grads = [], [], []
    try:
        for u in range(U):
            for i in f["insert_order"]:
                if int(f["versions"][i]) != u:
                    continue
                sid = SampleId(str(f["ids"][i]), int(f["turns"][i]), int(f["trajs"][i]))
                store.insert(agent, u, sid)
                store.set_cell_payload(agent, sid, u, "prompt", payload(f, int(f["prompt_off"][i])))
                store.set_cell_payload(agent, sid, u, "response", payload(f, int(f["resp_off"][i])))
                store.set_cell(agent, sid, u, "advantage", float(f["adv"][i]))
            for _ in range(G // mb):
                batch = store.poll_micro_batch(agent, u, mb)
                assert batch is not None
                polled += [key_to_idx[(r.sample_id.input_id, r.sample_id.number_of_turns,
                                       r.sample_id.trajectory_id, r.policy_version)] for r in batch.samples]
                reports = []
                eng.train_micro_batch(agent, batch, schema, reports.append)
                eng.run()
                if hooks and "after_mb" in hooks:
                    hooks["after_mb"](eng, agent, batch)
                store.complete(agent, batch.samples)
                mbn.append(reports[0].grad_norm)
            grads.append(eng.read_grad(agent))
            eng.apply_global_update(agent)
        st = eng.peek_state(agent)
        return dict(poll_order=np.array(polled), mb_grad_norm=np.array(mbn),
                    upd_grad_norm=np.array(eng.update_grad_norms[agent]), W=st.weights, m=st.m, v=st.v,
                    grads=grads, engine=eng)
    finally:
        store.close()
        eng.close()
