"""oracle/store_oracle.py — TEST INFRASTRUCTURE ONLY (the parity checker, never the product).

Pure-Python restatement of the reference experience-store lifecycle, used to
pin the golden store scripts (tests/golden/store_script_*.txt) and to check the
on-device table (fm_dtable) against them:

  * ExperienceStore::insert / set_cell / set_cell_payload / poll_micro_batch /
    purge_stale / complete / purge_inputs / drop_record / ready_count /
    record_count  (experience_store.hpp:44-191), canonical std::map order over
    (input_id, turns, traj, version) (experience_store.hpp:242-247)
  * RolloutEngine::release_group (rollout.hpp:812-834) with rule_reward and
    group_advantages (training.hpp:54-83), evaluated in the reference's
    sequential order so the doubles are bit-identical.

Script format and result lines: see ref_store_script in oracle/ref_driver.cpp.
Error lines carry fm_status = marlsim::ErrorCode + 1.
"""
from __future__ import annotations

import math

COLUMNS = [("prompt", "List"), ("response", "List"), ("logprobs", "Tensor"),
           ("reward", "Float"), ("advantage", "Float")]
BY_VALUE = {"Int", "Float", "Bool"}

# fm_status codes (marlsim::ErrorCode + 1, errors.hpp:10-39)
DUPLICATE_SAMPLE, UNKNOWN_COLUMN, RECORD_NOT_FOUND, CELL_ALREADY_SET = 12, 13, 14, 15
NOT_PROCESSING, BAD_SAMPLE_ID, CONFIG_ERROR = 17, 18, 26
DUPLICATE_KEY = 5


class StoreError(Exception):
    def __init__(self, code: int):
        super().__init__(code)
        self.code = code


def rule_reward(resp, pat) -> float:  # training.hpp:71-83
    if not resp or not pat:
        return 0.0
    best = 0
    for start in range(len(resp)):
        ln = 0
        while ln < len(pat) and start + ln < len(resp) and resp[start + ln] == pat[ln]:
            ln += 1
        best = max(best, ln)
    return best / len(pat)


def group_advantages(rewards, eps=1e-8):  # training.hpp:54-67, same operation order
    if not rewards:
        return []
    mean = 0.0
    for r in rewards:
        mean += r
    mean /= len(rewards)
    var = 0.0
    for r in rewards:
        var += (r - mean) * (r - mean)
    var /= len(rewards)
    sd = math.sqrt(var)
    return [(r - mean) / (sd + eps) for r in rewards]


class OracleStore:
    """One table with the orchestrator schema (orchestrator.hpp:191-195)."""

    def __init__(self):
        self.recs = {}  # key (id, t, j, v) -> {"cells": {}, "processing": bool}

    def insert(self, v, sid):  # experience_store.hpp:44-59
        if not sid[0] or "_" in sid[0]:
            raise StoreError(BAD_SAMPLE_ID)
        key = (*sid, v)
        if key in self.recs:
            raise StoreError(DUPLICATE_SAMPLE)
        self.recs[key] = {"cells": {}, "processing": False}

    def set_cell(self, v, sid, col, value, by_value=True):  # experience_store.hpp:61-80
        types = dict(COLUMNS)
        if col not in types:
            raise StoreError(UNKNOWN_COLUMN)
        rec = self.recs.get((*sid, v))
        if rec is None:
            raise StoreError(RECORD_NOT_FOUND)
        if col in rec["cells"]:
            # set_cell_payload registers the object first (experience_store.hpp:86): its
            # sample-field key already exists -> DuplicateKey (object_store.hpp:144-148)
            raise StoreError(DUPLICATE_KEY if not by_value and types[col] not in BY_VALUE else CELL_ALREADY_SET)
        if (types[col] in BY_VALUE) != by_value:
            raise StoreError(CONFIG_ERROR)
        rec["cells"][col] = value

    def _ready(self, rec):
        return len(rec["cells"]) == len(COLUMNS)

    def poll(self, v, mb):  # experience_store.hpp:92-114
        if mb < 1:
            raise StoreError(CONFIG_ERROR)
        chosen = []
        for key in sorted(self.recs):
            rec = self.recs[key]
            if rec["processing"] or key[3] != v or not self._ready(rec):
                continue
            chosen.append(key)
            if len(chosen) == mb:
                break
        if len(chosen) < mb:
            return None
        for k in chosen:
            self.recs[k]["processing"] = True
        return chosen

    def complete(self, keys):  # experience_store.hpp:134-148
        for k in keys:
            if k not in self.recs or not self.recs[k]["processing"]:
                raise StoreError(NOT_PROCESSING)
        for k in keys:
            del self.recs[k]

    def purge(self, pred):
        gone = [k for k, r in self.recs.items() if not r["processing"] and pred(k)]
        for k in gone:
            del self.recs[k]
        return len(gone)

    def drop(self, key):  # experience_store.hpp:166-175
        r = self.recs.get(key)
        if r is None or r["processing"]:
            return False
        del self.recs[key]
        return True

    def ready(self, v):
        return sum(1 for k, r in self.recs.items() if not r["processing"] and k[3] == v and self._ready(r))


def hexf(x: float) -> str:
    """printf("%a") of a double, as the reference driver prints it."""
    if x == 0.0:
        return "-0x0p+0" if math.copysign(1.0, x) < 0 else "0x0p+0"
    h = float.hex(x)  # e.g. '0x1.8000000000000p-1' -> strip trailing zeros like glibc
    sign = "-" if h.startswith("-") else ""
    h = h.lstrip("-")
    mant, exp = h[2:].split("p")
    if "." in mant:
        mant = mant.rstrip("0").rstrip(".")
    e = int(exp)
    return f"{sign}0x{mant}p{'+' if e >= 0 else '-'}{abs(e)}"


def replay(script: str, store=None) -> str:
    """Replay a script on the oracle (or on any object with the same adapter
    methods, e.g. the device-table adapter in tests/store_script.py)."""
    st = store if store is not None else OracleAdapter()
    out = []
    for line in script.splitlines():
        if not line.strip():
            continue
        f = line.split()
        op, a = f[0], f[1:]
        try:
            out.append(st.op(op, a))
        except StoreError as e:
            out.append(f"err {e.code}")
    return "\n".join(out) + "\n"


def parse_release(a):
    eps = float.fromhex(a[0]) if a[0].startswith(("0x", "-0x")) else float(a[0])
    np_ = int(a[1])
    pat = [int(x) for x in a[2:2 + np_]]
    i = 2 + np_
    ns = int(a[i]); i += 1
    surv = []
    for _ in range(ns):
        v, sid, t, j, nrec = int(a[i]), a[i + 1], int(a[i + 2]), int(a[i + 3]), int(a[i + 4]); i += 5
        recs = []
        for _ in range(nrec):
            recs.append((a[i + 1], int(a[i + 2]), int(a[i + 3]), int(a[i])))
            i += 4
        surv.append(((sid, t, j, v), recs))
    return eps, pat, surv


class OracleAdapter:
    def __init__(self):
        self.s = OracleStore()
        self.responses = {}

    def op(self, op, a):
        s = self.s
        if op == "insert":
            s.insert(int(a[0]), (a[1], int(a[2]), int(a[3])))
            return "ok"
        if op == "setf":
            s.set_cell(int(a[0]), (a[1], int(a[2]), int(a[3])), a[4], float.fromhex(a[5]), True)
            return "ok"
        if op == "setp":
            toks = [int(x) for x in a[6:6 + int(a[5])]]
            s.set_cell(int(a[0]), (a[1], int(a[2]), int(a[3])), a[4], toks, False)
            if a[4] == "response":
                self.responses[(a[1], int(a[2]), int(a[3]), int(a[0]))] = toks
            return "ok"
        if op == "poll":
            keys = s.poll(int(a[0]), int(a[1]))
            if keys is None:
                return "none"
            return " ".join(f"{k[0]}_{k[1]}_{k[2]}@{k[3]}:{hexf(s.recs[k]['cells']['advantage'])}" for k in keys)
        if op == "complete":
            k = int(a[0])
            keys = [(a[2 + 4 * i], int(a[3 + 4 * i]), int(a[4 + 4 * i]), int(a[1 + 4 * i])) for i in range(k)]
            s.complete(keys)
            return "ok"
        if op == "purge_stale":
            v = int(a[0])
            return str(s.purge(lambda k: k[3] < v))
        if op == "purge_inputs":
            ids = set(a[1:1 + int(a[0])])
            return str(s.purge(lambda k: k[0] in ids))
        if op == "drop":
            return "1" if s.drop((a[1], int(a[2]), int(a[3]), int(a[0]))) else "0"
        if op == "ready":
            return str(s.ready(int(a[0])))
        if op == "count":
            return str(len(s.recs))
        if op == "release":
            eps, pat, surv = parse_release(a)
            rewards = [rule_reward(self.responses[k], pat) for k, _ in surv]
            advs = group_advantages(rewards, eps)
            for (k, recs), r, ad in zip(surv, rewards, advs):
                for (sid, t, j, v) in recs:
                    s.set_cell(v, (sid, t, j), "reward", r)
                    s.set_cell(v, (sid, t, j), "advantage", ad)
            return " ".join(f"{hexf(r)}/{hexf(ad)}" for r, ad in zip(rewards, advs)) or "ok"
        return "bad-op"
