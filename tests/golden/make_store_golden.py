"""Generates tests/golden/store_script_*.txt (+ .expected) from the COMPILED
REFERENCE ExperienceStore (oracle/_ref, ref_store_script in oracle/ref_driver.cpp).

    python tests/golden/make_store_golden.py

A script is a seeded random lifecycle of one agent table over several policy
versions: GRPO groups inserted in shuffled input order, prompt/response/logprob
payloads, group releases (rule_reward + group_advantages, rollout.hpp:812-834)
over survivors after random drops, polls of the canonical-first ready records,
completes, purge_stale at version bumps, purge_inputs, and the reference's
error paths (duplicate insert, bad ids, double set, unknown column, storage
class mismatch, completing unpolled records, mb < 1).  The .expected file is
the reference's own output; tests/test_store_oracle.py pins the Python
restatement against it and tests/test_gpu_dtable.py the device table.
"""
from __future__ import annotations

import random
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as orc  # noqa: E402

OUT = Path(__file__).resolve().parent
PATTERN = [3, 1, 4]


def make_script(seed: int, versions: int = 4, groups_per_version: int = 6, k: int = 4, mb: int = 4,
                vocab: int = 8) -> str:
    rng = random.Random(seed)
    lines = []
    polled = []  # (v, id, t, j) currently processing
    ids_pool = [f"q{n:05d}" for n in rng.sample(range(200), 40)] + ["a", "zz", "q1", "b7"]
    for v in range(versions):
        ids = rng.sample(ids_pool, groups_per_version)
        groups = []
        for gid in ids:
            trajs = list(range(k))
            rng.shuffle(trajs)
            recs = []
            for j in trajs:
                turns = 0 if rng.random() < 0.8 else 1
                lines.append(f"insert {v} {gid} {turns} {j}")
                plen = rng.randint(1, 6)
                lines.append(f"setp {v} {gid} {turns} {j} prompt {plen} " +
                             " ".join(str(rng.randrange(vocab)) for _ in range(plen)))
                recs.append((gid, turns, j))
            groups.append((gid, recs))
        # error paths, interleaved
        g0, r0 = groups[0][0], groups[0][1][0]
        lines.append(f"insert {v} {g0} {r0[1]} {r0[2]}")              # DuplicateSample
        lines.append(f"insert {v} bad_id 0 0")                         # BadSampleId
        lines.append(f"setf {v} {g0} {r0[1]} {r0[2]} nosuch 0x1p+0")   # UnknownColumn
        lines.append(f"setf {v} {g0} {r0[1]} {r0[2]} prompt 0x1p+0")   # storage-class mismatch
        lines.append(f"setf {v} zz9 0 0 reward 0x1p+0")                # RecordNotFound
        lines.append(f"setp {v} {g0} {r0[1]} {r0[2]} prompt 1 5")      # CellAlreadySet
        lines.append(f"poll {v} 0")                                    # ConfigError
        lines.append(f"setp {v} {g0} {r0[1]} {r0[2]} advantage 1 5")   # payload into a by-value column
        # responses (some contain the reward pattern), logprobs
        order = [(g, r) for g, recs in groups for r in recs]
        rng.shuffle(order)
        for g, (gid, t, j) in order:
            n = rng.randint(0, 12)
            toks = [rng.randrange(vocab) for _ in range(n)]
            if n >= 3 and rng.random() < 0.5:
                p = rng.randrange(n - 2)
                ln = rng.randint(1, 3)
                toks[p:p + ln] = PATTERN[:ln]
            lines.append(f"setp {v} {gid} {t} {j} response {len(toks)} " + " ".join(map(str, toks)))
            lines.append(f"setp {v} {gid} {t} {j} logprobs 1 0")
            if rng.random() < 0.3:
                lines.append(f"ready {v}")
        # drops, then release every group over its survivors
        for gid, recs in groups:
            surv = list(recs)
            if rng.random() < 0.3:
                d = surv.pop(rng.randrange(len(surv)))
                lines.append(f"drop {v} {gid} {d[1]} {d[2]}")
                lines.append(f"drop {v} {gid} {d[1]} {d[2]}")  # already gone -> 0
            parts = [f"release 0x1.5798ee2308c3ap-27 3 {' '.join(map(str, PATTERN))} {len(surv)}"]
            for (g, t, j) in surv:
                parts.append(f"{v} {g} {t} {j} 1 {v} {g} {t} {j}")
            lines.append(" ".join(parts))
        lines.append(f"ready {v}")
        lines.append("count")
        lines.append(f"setp {v} {g0} {r0[1]} {r0[2]} reward 1 5")      # by-value cell already set
        lines.append(f"setf {v} {g0} {r0[1]} {r0[2]} response 0x1p+0")  # ref cell already set
        # polls and completes
        for _ in range(rng.randint(2, 5)):
            lines.append(f"poll {v} {mb}")
            lines.append("__COMPLETE_LAST__" if rng.random() < 0.6 else "__HOLD__")
        lines.append(f"poll {v} 64")                                   # too few ready -> nullopt
        if v >= 1:
            lines.append(f"poll {v - 1} 2")                            # an older version's leftovers
        lines.append(f"complete 1 {v} {groups[-1][0]} 0 99")  # NotProcessing
        if v >= 1:
            lines.append(f"purge_stale {v}")
        if rng.random() < 0.5:
            lines.append(f"purge_inputs 2 {rng.choice(ids_pool)} {ids[-1]}")
        lines.append("count")
    return "\n".join(lines) + "\n"


def resolve(script: str) -> str:
    """Turns the __COMPLETE_LAST__ markers into explicit completes of the records
    the preceding poll returned (per the reference's own answer)."""
    out = []
    for line in script.splitlines():
        if line in ("__COMPLETE_LAST__", "__HOLD__"):
            if line == "__COMPLETE_LAST__":
                res = orc.ref_store_script("\n".join(out) + "\n").splitlines()[-1]
                if res not in ("none",) and not res.startswith("err"):
                    keys = [tok.split(":")[0] for tok in res.split()]
                    parts = []
                    for k in keys:
                        sid, v = k.split("@")
                        gid, t, j = sid.rsplit("_", 2)
                        parts.append(f"{v} {gid} {t} {j}")
                    out.append(f"complete {len(parts)} " + " ".join(parts))
            continue
        out.append(line)
    return "\n".join(out) + "\n"


def main():
    for seed in (1, 2, 3):
        script = resolve(make_script(seed))
        (OUT / f"store_script_{seed}.txt").write_text(script)
        (OUT / f"store_script_{seed}.expected").write_text(orc.ref_store_script(script))
        print(seed, len(script.splitlines()), "ops")


if __name__ == "__main__":
    main()
