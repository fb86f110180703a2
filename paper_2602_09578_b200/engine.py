"""Host-side mirror of the reference's hot-path interfaces over the C ABI.

Same class and method names, argument meaning and error behaviour as
  * ``marlsim::ExperienceStore``  (experience_store.hpp:19-276)
  * ``marlsim::TrainingEngine``   (training.hpp:192-540)
  * ``marlsim::group_advantages`` (training.hpp:54-67)
so that parity tests read like the reference's own usage.  All compute goes
through ``libflexmarl_b200.so`` (tcgen05 / CUDA kernels); errors are raised
as :class:`MarlsimError` carrying the reference ``ErrorCode`` name.

Completion is asynchronous exactly as in the reference: ``train_micro_batch``
returns at once and its ``on_done(GradReport)`` fires from :meth:`run`
(the event-loop drain, sim.hpp:63-67), never inline.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib
from ._lib import FlexMarlError, check, lib, ptr

MarlsimError = FlexMarlError

COLUMN_TYPES = {"Int": 0, "Float": 1, "Bool": 2, "String": 3, "List": 4, "Tensor": 5}


# ---------------------------------------------------------------------------
# value types (sample.hpp)
# ---------------------------------------------------------------------------
@dataclass(frozen=True, order=True)
class SampleId:
    input_id: str
    number_of_turns: int = 0
    trajectory_id: int = 0

    def render(self) -> str:  # sample.hpp:21-24
        return f"{self.input_id}_{self.number_of_turns}_{self.trajectory_id}"


@dataclass
class TableSchema:
    agent_id: str
    columns: list  # [(name, type-name)]

    def column_index(self, name: str) -> int:
        for i, (n, _) in enumerate(self.columns):
            if n == name:
                return i
        return -1


@dataclass
class SampleRecord:
    policy_version: int
    sample_id: SampleId
    handle: int
    cell: _lib.fm_sample  # arena offsets of prompt/response + advantage


@dataclass
class MicroBatch:
    agent_id: str
    policy_version: int
    samples: list = field(default_factory=list)
    # set when polled from a DeviceExperienceStore: the descriptors stay in HBM
    dtable: object = None
    poll_id: int = -1
    rows: int = 0

    def size(self) -> int:
        return len(self.samples)


@dataclass
class GradReport:  # training.hpp:169-177
    agent_id: str
    batch_version: int
    engine_version: int
    batch_size: int
    grad_norm: float
    tokens: int = 0
    loss: float = 0.0


@dataclass
class AdamParams:  # training.hpp:24-29
    lr: float = 1e-6
    beta1: float = 0.9
    beta2: float = 0.999
    eps: float = 1e-8


@dataclass
class PolicyState:
    agent_id: str
    version: int
    step_count: int
    samples_accumulated: int
    weights: np.ndarray
    m: np.ndarray
    v: np.ndarray


# ---------------------------------------------------------------------------
# device context
# ---------------------------------------------------------------------------
class Context:
    """One GPU (fm_ctx): compute + two copy streams, token arena, workspace."""

    def __init__(self, device: int = 0):
        self._h = C.c_void_p()
        check(lib().fm_ctx_create(device, C.byref(self._h)))
        self.device = device

    @property
    def handle(self):
        return self._h

    @property
    def num_sms(self) -> int:
        return lib().fm_ctx_num_sms(self._h)

    def reserve(self, arena_bytes: int, max_rows: int = 0, vocab: int = 0, feat: int = 0) -> None:
        check(lib().fm_ctx_reserve(self._h, arena_bytes, max_rows, vocab, feat))

    def put(self, payload: bytes) -> int:
        off = C.c_uint64()
        buf = (C.c_uint8 * len(payload)).from_buffer_copy(payload)
        check(lib().fm_arena_put(self._h, buf, len(payload), C.byref(off)))
        return off.value

    def reset_arena(self) -> None:
        check(lib().fm_arena_reset(self._h))

    def synchronize(self) -> None:
        check(lib().fm_ctx_synchronize(self._h))

    def close(self) -> None:
        if self._h:
            lib().fm_ctx_destroy(self._h)
            self._h = C.c_void_p()


def group_advantages(ctx: Context, rewards, seg_off=None, eps_adv: float = 1e-8) -> np.ndarray:
    """training.hpp:54-67 on the device (K-adv).  Without seg_off the whole
    list is one group, as in the reference signature."""
    r = np.ascontiguousarray(rewards, dtype=np.float64)
    if seg_off is None:
        seg_off = np.array([0, len(r)], dtype=np.int32)
    off = np.ascontiguousarray(seg_off, dtype=np.int32)
    out = np.zeros_like(r)
    if len(r) == 0:
        return out
    check(lib().fm_group_advantages(ctx.handle, ptr(r), ptr(off), len(off) - 1, eps_adv, ptr(out)))
    return out


def seeded_weights(vocab: int, feat: int, seed: int, threads: int = 0) -> np.ndarray:
    """PolicyModel::seeded (policy.hpp:29-35), bit-identical, on the host."""
    w = np.empty(vocab * feat, dtype=np.float64)
    check(lib().fm_seeded_weights(vocab, feat, seed, ptr(w), threads))
    return w.reshape(vocab, feat)


def agent_seed(seed: int, agent: str) -> int:
    return lib().fm_agent_seed(seed, agent.encode())


# ---------------------------------------------------------------------------
# experience store (experience_store.hpp)
# ---------------------------------------------------------------------------
class ExperienceStore:
    def __init__(self, ctx: Context):
        self._h = C.c_void_p()
        check(lib().fm_store_create(C.byref(self._h)))
        self.ctx = ctx
        self._schemas: dict[str, TableSchema] = {}

    def create_table(self, schema: TableSchema) -> None:
        names = [n.encode() for n, _ in schema.columns]
        arr = (C.c_char_p * len(names))(*names)
        types = (C.c_int * len(names))(*[COLUMN_TYPES[t] for _, t in schema.columns])
        check(lib().fm_store_create_table(self._h, schema.agent_id.encode(), arr, types, len(names)))
        self._schemas[schema.agent_id] = schema

    def has_table(self, agent_id: str) -> bool:
        return agent_id in self._schemas

    def schema(self, agent_id: str) -> TableSchema:
        if agent_id not in self._schemas:
            raise MarlsimError(16, agent_id)
        return self._schemas[agent_id]

    def insert(self, agent_id: str, policy_version: int, sid: SampleId) -> None:
        check(lib().fm_store_insert(self._h, agent_id.encode(), policy_version, sid.input_id.encode(),
                                    sid.number_of_turns, sid.trajectory_id))

    def set_cell(self, agent_id: str, sid: SampleId, version: int, column: str, value: float) -> None:
        check(lib().fm_store_set_float(self._h, agent_id.encode(), sid.input_id.encode(),
                                       sid.number_of_turns, sid.trajectory_id, version,
                                       column.encode(), float(value)))

    def set_cell_payload(self, agent_id: str, sid: SampleId, version: int, column: str,
                         payload: bytes) -> None:
        buf = (C.c_uint8 * len(payload)).from_buffer_copy(payload)
        check(lib().fm_store_set_payload(self._h, self.ctx.handle, agent_id.encode(),
                                         sid.input_id.encode(), sid.number_of_turns, sid.trajectory_id,
                                         version, column.encode(), buf, len(payload)))

    def ready_count(self, agent_id: str, version: int) -> int:
        out = C.c_uint64()
        check(lib().fm_store_ready_count(self._h, agent_id.encode(), version, C.byref(out)))
        return out.value

    def record_count(self, agent_id: str) -> int:
        out = C.c_uint64()
        check(lib().fm_store_record_count(self._h, agent_id.encode(), C.byref(out)))
        return out.value

    def poll_micro_batch(self, agent_id: str, current_version: int, micro_batch_size: int,
                         columns=("prompt", "response", "advantage")) -> Optional[MicroBatch]:
        n = int(micro_batch_size)
        samples = (_lib.fm_sample * max(n, 1))()
        handles = (C.c_int64 * max(n, 1))()
        got = C.c_int64()
        pc, rc, ac = (c.encode() if c else None for c in (columns or (None, None, None)))
        check(lib().fm_store_poll(self._h, agent_id.encode(), current_version, n, pc, rc, ac,
                                  samples if pc else None, handles, C.byref(got)))
        if got.value == 0:
            return None
        batch = MicroBatch(agent_id, current_version)
        idbuf = C.create_string_buffer(256)
        turns, traj, ver = C.c_int(), C.c_int(), C.c_int64()
        for i in range(n):
            check(lib().fm_store_record_id(self._h, agent_id.encode(), handles[i], idbuf, 256,
                                           C.byref(turns), C.byref(traj), C.byref(ver)))
            batch.samples.append(SampleRecord(ver.value, SampleId(idbuf.value.decode(), turns.value, traj.value),
                                              handles[i], _lib.fm_sample(samples[i].prompt_off,
                                                                         samples[i].response_off,
                                                                         samples[i].advantage)))
        return batch

    def complete(self, agent_id: str, samples: list) -> None:
        hs = (C.c_int64 * max(len(samples), 1))(*[s.handle for s in samples])
        check(lib().fm_store_complete(self._h, agent_id.encode(), hs, len(samples)))

    def purge_stale(self, agent_id: str, current_version: int) -> int:
        out = C.c_uint64()
        check(lib().fm_store_purge_stale(self._h, agent_id.encode(), current_version, C.byref(out)))
        return out.value

    def close(self) -> None:
        if self._h:
            lib().fm_store_destroy(self._h)
            self._h = C.c_void_p()


# ---------------------------------------------------------------------------
# on-device experience store (experience_store.hpp, rollout.hpp:812-834)
# ---------------------------------------------------------------------------
def _ids(strings):
    enc = [x.encode() for x in strings]
    return (C.c_char_p * max(len(enc), 1))(*enc)


class DeviceExperienceStore:
    """ExperienceStore whose tables live in one GPU's HBM (fm_dtable).

    Same methods and error behaviour as :class:`ExperienceStore`; records are
    also addressable by their slot (``find``).  Two rollout-side entry points
    keep the producer on the device too: :meth:`generate` (rollout completion,
    rollout.hpp:715-731) and :meth:`release_groups` (rollout.hpp:812-834).
    """

    def __init__(self, ctx: Context, capacity: int = 4096):
        self.ctx = ctx
        self.capacity = capacity
        self._t: dict[str, C.c_void_p] = {}
        self._schemas: dict[str, TableSchema] = {}

    def _h(self, agent_id: str):
        if agent_id not in self._t:
            raise MarlsimError(16, agent_id)  # UnknownTable
        return self._t[agent_id]

    def create_table(self, schema: TableSchema, capacity: int | None = None) -> None:
        if schema.agent_id in self._t:
            raise MarlsimError(10, schema.agent_id)  # TableExists
        names = [n.encode() for n, _ in schema.columns]
        arr = (C.c_char_p * max(len(names), 1))(*names)
        types = (C.c_int * max(len(names), 1))(*[COLUMN_TYPES[t] for _, t in schema.columns])
        h = C.c_void_p()
        check(lib().fm_dtable_create(self.ctx.handle, schema.agent_id.encode(), arr, types, len(names),
                                     capacity or self.capacity, C.byref(h)))
        self._t[schema.agent_id] = h
        self._schemas[schema.agent_id] = schema

    def has_table(self, agent_id: str) -> bool:
        return agent_id in self._t

    def schema(self, agent_id: str) -> TableSchema:
        self._h(agent_id)
        return self._schemas[agent_id]

    def table(self, agent_id: str):
        return self._h(agent_id)

    def insert(self, agent_id: str, policy_version: int, sid: SampleId) -> int:
        return int(self.insert_many(agent_id, policy_version, [sid])[0])

    def insert_many(self, agent_id: str, policy_version: int, sids) -> np.ndarray:
        sids = list(sids)
        out = np.zeros(max(len(sids), 1), np.int64)
        turns = np.array([s.number_of_turns for s in sids] or [0], np.int32)
        trajs = np.array([s.trajectory_id for s in sids] or [0], np.int32)
        check(lib().fm_dtable_insert(self._h(agent_id), policy_version, len(sids), _ids([s.input_id for s in sids]),
                                     ptr(turns), ptr(trajs), ptr(out)))
        return out[:len(sids)]

    def find(self, agent_id: str, sid: SampleId, version: int) -> int:
        out = C.c_int64()
        check(lib().fm_dtable_find(self._h(agent_id), sid.input_id.encode(), sid.number_of_turns,
                                   sid.trajectory_id, version, C.byref(out)))
        return out.value

    def _slot(self, agent_id: str, sid: SampleId, version: int) -> int:
        s = self.find(agent_id, sid, version)
        if s < 0:
            raise MarlsimError(14, sid.render())  # RecordNotFound
        return s

    def set_cell(self, agent_id: str, sid: SampleId, version: int, column: str, value: float) -> None:
        self.set_cells(agent_id, column, [self._slot(agent_id, sid, version)], [value])

    def set_cells(self, agent_id: str, column: str, slots, values) -> None:
        sl = np.ascontiguousarray(slots, np.int64)
        vals = np.ascontiguousarray(values, np.float64)
        check(lib().fm_dtable_set_float(self._h(agent_id), column.encode(), len(sl), ptr(sl), ptr(vals)))

    def set_cell_payload(self, agent_id: str, sid: SampleId, version: int, column: str, payload: bytes) -> None:
        self.set_payload_slot(agent_id, column, self._slot(agent_id, sid, version), payload)

    def set_payload_slot(self, agent_id: str, column: str, slot: int, payload: bytes) -> None:
        buf = (C.c_uint8 * len(payload)).from_buffer_copy(payload)
        check(lib().fm_dtable_set_payload(self._h(agent_id), column.encode(), slot, buf, len(payload)))

    def generate(self, agent_id: str, weights, slots, prompts, max_tokens: int, seeds,
                 response_col: str = "response", logprob_col: str | None = "logprobs") -> None:
        """Rollout completion on the GPU: PolicyModel::generate per record, the
        responses (and log-probs) written straight into the arena and the cells."""
        sl = np.ascontiguousarray(slots, np.int64)
        off = np.zeros(len(prompts) + 1, np.int32)
        off[1:] = np.cumsum([len(p) for p in prompts])
        flat = np.ascontiguousarray(np.concatenate([np.asarray(p, np.int32) for p in prompts])
                                    if off[-1] else np.zeros(1, np.int32), np.int32)
        sd = np.ascontiguousarray(seeds, np.uint64)
        check(lib().fm_dtable_generate(self._h(agent_id), weights, response_col.encode(),
                                       logprob_col.encode() if logprob_col else None, len(sl), ptr(sl),
                                       ptr(flat), ptr(off), max_tokens, ptr(sd)))

    def release_groups(self, groups, pattern=(3, 1, 4), eps_adv: float = 1e-8, response_col: str = "response",
                       reward_col: str = "reward", adv_col: str = "advantage", read_back: bool = False):
        """release_group (rollout.hpp:812-834) for several groups at once.  A group
        is a list of survivors; a survivor is ``(score, records)`` with ``score`` =
        (agent, slot) of the record whose response is scored and ``records`` the
        (agent, slot) list that receives reward and advantage."""
        agents = []
        for grp in groups:
            for (sa, _), recs in grp:
                for a in [sa] + [r[0] for r in recs]:
                    if a not in agents:
                        agents.append(a)
        tix = {a: i for i, a in enumerate(agents)}
        seg = [0]
        st, ss, ro, rt, rs = [], [], [0], [], []
        for grp in groups:
            for (sa, sslot), recs in grp:
                st.append(tix[sa])
                ss.append(sslot)
                for a, slot in recs:
                    rt.append(tix[a])
                    rs.append(slot)
                ro.append(len(rs))
            seg.append(len(st))
        tabs = (C.c_void_p * len(agents))(*[self._h(a).value for a in agents])
        arrs = [np.ascontiguousarray(x, dt) if len(x) else np.zeros(1, dt) for x, dt in
                ((seg, np.int32), (st, np.int32), (ss, np.int64), (ro, np.int32), (rt, np.int32), (rs, np.int64))]
        pat = np.ascontiguousarray(pattern if len(pattern) else [0], np.int32)
        n = len(st)
        rew = np.zeros(max(n, 1))
        adv = np.zeros(max(n, 1))
        check(lib().fm_dtable_release_groups(tabs, len(agents), response_col.encode(), reward_col.encode(),
                                             adv_col.encode(), len(groups), *[ptr(a) for a in arrs], ptr(pat),
                                             len(pattern), eps_adv, ptr(rew) if read_back else None,
                                             ptr(adv) if read_back else None))
        return (rew[:n], adv[:n]) if read_back else None

    def ready_count(self, agent_id: str, version: int) -> int:
        out = C.c_uint64()
        check(lib().fm_dtable_ready_count(self._h(agent_id), version, C.byref(out)))
        return out.value

    def record_count(self, agent_id: str) -> int:
        out = C.c_uint64()
        check(lib().fm_dtable_record_count(self._h(agent_id), C.byref(out)))
        return out.value

    def record(self, agent_id: str, slot: int) -> SampleRecord:
        idbuf = C.create_string_buffer(4096)
        turns, traj, ver, proc, st = C.c_int(), C.c_int(), C.c_int64(), C.c_int(), C.c_uint32()
        check(lib().fm_dtable_record(self._h(agent_id), slot, idbuf, 4096, C.byref(turns), C.byref(traj),
                                     C.byref(ver), C.byref(proc), C.byref(st)))
        return SampleRecord(ver.value, SampleId(idbuf.value.decode(), turns.value, traj.value), slot, None)

    def poll_micro_batch(self, agent_id: str, current_version: int, micro_batch_size: int,
                         columns=("prompt", "response", "advantage")) -> Optional[MicroBatch]:
        n = int(micro_batch_size)
        slots = np.zeros(max(n, 1), np.int64)
        rows, got, pid = C.c_int64(), C.c_int64(), C.c_int64()
        pc, rc, ac = (c.encode() if c else None for c in (columns or (None, None, None)))
        check(lib().fm_dtable_poll(self._h(agent_id), current_version, n, pc, rc, ac, ptr(slots),
                                   C.byref(rows), C.byref(got), C.byref(pid)))
        if got.value == 0:
            return None
        batch = MicroBatch(agent_id, current_version, dtable=self._h(agent_id), poll_id=pid.value,
                           rows=rows.value)
        cap = 256
        ids = C.create_string_buffer(n * cap)
        turns, trajs, vers = np.zeros(n, np.int32), np.zeros(n, np.int32), np.zeros(n, np.int64)
        check(lib().fm_dtable_records(self._h(agent_id), n, ptr(slots), ids, cap, ptr(turns), ptr(trajs), ptr(vers)))
        raw = ids.raw
        batch.samples = [SampleRecord(int(vers[i]), SampleId(raw[i * cap:(i + 1) * cap].split(b"\0", 1)[0].decode(),
                                                             int(turns[i]), int(trajs[i])), int(slots[i]), None)
                         for i in range(n)]
        if any(len(s.sample_id.input_id) >= cap - 1 for s in batch.samples):  # long ids: one query each
            batch.samples = [self.record(agent_id, int(s)) for s in slots[:n]]
        return batch

    def read_cells(self, agent_id: str, column: str, slots, as_float: bool = True) -> np.ndarray:
        sl = np.ascontiguousarray(slots, np.int64)
        out = np.zeros(max(len(sl), 1), np.uint64)
        check(lib().fm_dtable_read_cells(self._h(agent_id), column.encode(), len(sl), ptr(sl), ptr(out)))
        out = out[:len(sl)]
        return out.view(np.float64) if as_float else out

    def complete(self, agent_id: str, samples: list) -> None:
        hs = np.ascontiguousarray([s.handle for s in samples] or [0], np.int64)
        check(lib().fm_dtable_complete(self._h(agent_id), ptr(hs), len(samples)))

    def purge_stale(self, agent_id: str, current_version: int) -> int:
        out = C.c_uint64()
        check(lib().fm_dtable_purge_stale(self._h(agent_id), current_version, C.byref(out)))
        return out.value

    def purge_inputs(self, agent_id: str, inputs) -> int:
        inputs = list(inputs)
        out = C.c_uint64()
        check(lib().fm_dtable_purge_inputs(self._h(agent_id), _ids(inputs), len(inputs), C.byref(out)))
        return out.value

    def drop_record(self, agent_id: str, sid: SampleId, version: int) -> bool:
        out = C.c_int()
        check(lib().fm_dtable_drop_record(self._h(agent_id), sid.input_id.encode(), sid.number_of_turns,
                                          sid.trajectory_id, version, C.byref(out)))
        return bool(out.value)

    def close(self) -> None:
        for h in self._t.values():
            lib().fm_dtable_destroy(h)
        self._t.clear()


# ---------------------------------------------------------------------------
# training engine (training.hpp)
# ---------------------------------------------------------------------------
@dataclass
class _Group:
    vocab: int
    feat: int
    handle: C.c_void_p = None
    ctx: Optional[Context] = None
    last_ctx: Optional[Context] = None
    in_flight: bool = False
    ever_ran: bool = False


class TrainingEngine:
    """Agent-centric trainer over a pool of GPU contexts (one agent per
    context at a time, STRICT_PACK of training.hpp:500-531 degenerates to
    'a free GPU, preferring the last one')."""

    def __init__(self, pool: list, global_batch: int = 64, adam: AdamParams | None = None,
                 seed: int = 2048, precision: int = _lib.PRECISION_BF16_TC, allowed_staleness: int = 0,
                 park_tier: int = _lib.TIER_DEVICE, slots_per_device: int = 1):
        self.pool = list(pool)
        self.global_batch = global_batch
        self.adam = adam or AdamParams()
        self.seed = seed
        self.precision = precision
        self.allowed_staleness = allowed_staleness
        self.park_tier = park_tier
        self.slots_per_device = slots_per_device
        self._groups: dict[str, _Group] = {}
        self._pending: list = []  # (agent, ticket, report-base, on_done)
        self.update_grad_norms: dict[str, list] = {}

    # -- registry ------------------------------------------------------------
    def add_agent(self, agent_id: str, vocab: int, feat: int) -> None:
        self._groups[agent_id] = _Group(vocab, feat)

    def _group(self, agent: str) -> _Group:
        if agent not in self._groups:
            raise MarlsimError(26, f"unknown agent {agent}")
        return self._groups[agent]

    def is_active(self, agent: str) -> bool:
        return self._group(agent).ctx is not None

    def in_flight(self, agent: str) -> bool:
        return self._group(agent).in_flight

    def param_count(self, agent: str) -> int:
        g = self._group(agent)
        return g.vocab * g.feat

    def initial_model(self, agent: str) -> np.ndarray:  # training.hpp:245-248
        g = self._group(agent)
        return seeded_weights(g.vocab, g.feat, agent_seed(self.seed, agent))

    def _free_ctx(self, agent: str) -> Optional[Context]:
        g = self._group(agent)
        used = {}
        for a, gg in self._groups.items():
            if gg.ctx is not None:
                used[id(gg.ctx)] = used.get(id(gg.ctx), 0) + 1
        free = [c for c in self.pool if used.get(id(c), 0) < self.slots_per_device]
        if not free:
            return None
        if g.last_ctx is not None and any(c is g.last_ctx for c in free):
            return g.last_ctx
        return free[0]

    def can_activate(self, agent: str) -> bool:
        return self._free_ctx(agent) is not None

    # -- lifecycle (training.hpp:259-350) -------------------------------------
    def activate(self, agent: str, on_done: Callable | None = None) -> None:
        g = self._group(agent)
        if g.ctx is not None:
            raise MarlsimError(26, f"{agent} already active")
        ctx = self._free_ctx(agent)
        if ctx is None:
            raise MarlsimError(21, f"no free training device for {agent}")
        if g.handle is None:
            h = C.c_void_p()
            check(lib().fm_agent_create(ctx.handle, agent.encode(), g.vocab, g.feat, self.precision, C.byref(h)))
            g.handle = h
            w0 = np.ascontiguousarray(self.initial_model(agent).reshape(-1))
            check(lib().fm_agent_set_weights(h, ptr(w0)))
        else:
            check(lib().fm_agent_activate(g.handle, ctx.handle))
        g.ctx = ctx
        g.last_ctx = ctx
        if on_done:
            self._pending.append((agent, None, None, on_done))

    def suspend(self, agent: str, on_done: Callable | None = None) -> None:
        g = self._group(agent)
        if g.ctx is None:
            raise MarlsimError(24, agent)
        if g.in_flight:
            raise MarlsimError(22, f"{agent} has a micro batch in flight")
        check(lib().fm_agent_suspend(g.handle, self.park_tier, -1))
        g.ctx = None
        if on_done:
            self._pending.append((agent, None, None, on_done))

    # -- hot path -------------------------------------------------------------
    def version(self, agent: str) -> int:
        g = self._group(agent)
        return 0 if g.handle is None else lib().fm_agent_version(g.handle)

    def train_micro_batch(self, agent: str, batch: MicroBatch, schema: TableSchema,
                          on_done: Callable | None = None) -> None:
        g = self._group(agent)
        if g.ctx is None:
            raise MarlsimError(24, agent)
        if g.in_flight:
            raise MarlsimError(22, agent)
        ver = lib().fm_agent_version(g.handle)
        staleness = ver - batch.policy_version
        if staleness < 0 or staleness > self.allowed_staleness:
            raise MarlsimError(23, f"{agent}: batch v{batch.policy_version} vs state v{ver}")
        if min(schema.column_index(c) for c in ("prompt", "response", "advantage")) < 0:
            raise MarlsimError(13, "trainer needs prompt/response/advantage columns")
        n = len(batch.samples)
        # DuplicateSample guard (training.hpp:396-401), before anything is enqueued
        ids = [s.sample_id.input_id.encode() for s in batch.samples]
        keys = (_lib.fm_sample_key * max(n, 1))(*[
            _lib.fm_sample_key(ids[i], s.sample_id.number_of_turns, s.sample_id.trajectory_id, s.policy_version)
            for i, s in enumerate(batch.samples)])
        check(lib().fm_agent_add_grad_keys(g.handle, keys, n))
        ticket = C.c_int64()
        if batch.dtable is not None:  # polled on the device: descriptors stay in HBM
            check(lib().fm_train_polled(g.handle, batch.dtable, batch.poll_id, self.global_batch, C.byref(ticket)))
        else:
            arr = (_lib.fm_sample * max(n, 1))(*[s.cell for s in batch.samples])
            check(lib().fm_train_micro_batch(g.handle, arr, n, self.global_batch, C.byref(ticket)))
        g.in_flight = True
        base = GradReport(agent, batch.policy_version, ver, n, float("nan"))
        self._pending.append((agent, ticket.value, base, on_done))

    def apply_global_update(self, agent: str) -> int:
        g = self._group(agent)
        if g.ctx is None:
            raise MarlsimError(24, agent)
        gn = C.c_double()
        ver = C.c_int64()
        a = self.adam
        check(lib().fm_apply_update(g.handle, self.global_batch, a.lr, a.beta1, a.beta2, a.eps,
                                    C.byref(gn), C.byref(ver)))
        self.update_grad_norms.setdefault(agent, []).append(gn.value)
        return ver.value

    def run(self) -> None:
        """Drain completions in submission order (the event-loop delivery)."""
        while self._pending:
            agent, ticket, base, cb = self._pending.pop(0)
            g = self._group(agent)
            if ticket is None:
                if g.ctx is not None:
                    check(lib().fm_agent_sync(g.handle))
                if cb:
                    cb()
                continue
            check(lib().fm_agent_sync(g.handle))
            rep = _lib.fm_report()
            r = lib().fm_agent_poll_report(g.handle, ticket, C.byref(rep))
            if r < 0 or r > 1:
                check(r)
            g.in_flight = False
            base.grad_norm = rep.grad_norm
            base.tokens = rep.tokens
            base.loss = rep.loss
            if cb:
                cb(base)

    def peek_state(self, agent: str) -> PolicyState:
        g = self._group(agent)
        if g.handle is None:
            raise MarlsimError(24, f"{agent} never ran")
        if g.ctx is None:
            raise MarlsimError(24, f"{agent} is suspended; activate to inspect")
        P = g.vocab * g.feat
        w = np.empty(P, dtype=np.float64)
        m = np.empty(P, dtype=np.float32)
        v = np.empty(P, dtype=np.float32)
        step = C.c_int64()
        check(lib().fm_agent_read_weights(g.handle, ptr(w)))
        check(lib().fm_agent_read_moments(g.handle, ptr(m), ptr(v), C.byref(step)))
        return PolicyState(agent, lib().fm_agent_version(g.handle), step.value,
                           lib().fm_agent_samples_accumulated(g.handle),
                           w.reshape(g.vocab, g.feat), m.reshape(g.vocab, g.feat), v.reshape(g.vocab, g.feat))

    def read_grad(self, agent: str) -> np.ndarray:
        g = self._group(agent)
        out = np.empty(g.vocab * g.feat, dtype=np.float64)
        check(lib().fm_agent_read_grad(g.handle, ptr(out)))
        return out.reshape(g.vocab, g.feat)

    def checksum(self, agent: str) -> int:
        out = C.c_uint64()
        check(lib().fm_agent_state_checksum(self._group(agent).handle, C.byref(out)))
        return out.value

    def handle(self, agent: str):
        return self._group(agent).handle

    def close(self) -> None:
        for g in self._groups.values():
            if g.handle is not None:
                lib().fm_agent_destroy(g.handle)
                g.handle = None
