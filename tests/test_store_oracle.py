"""CPU: the experience-store restatement (oracle/store_oracle.py) reproduces the
reference ExperienceStore lifecycle bit-for-bit on the golden scripts, and the
live compiled reference (oracle/_ref, when present) still produces the fixtures."""
from __future__ import annotations

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

from oracle import store_oracle as so  # noqa: E402
from oracle import oracle as orc  # noqa: E402

GOLD = ROOT / "tests" / "golden"
SEEDS = (1, 2, 3)


@pytest.mark.parametrize("seed", SEEDS)
def test_store_oracle_matches_reference_golden(seed):
    script = (GOLD / f"store_script_{seed}.txt").read_text()
    expected = (GOLD / f"store_script_{seed}.expected").read_text()
    assert so.replay(script) == expected


@pytest.mark.parametrize("seed", SEEDS)
def test_live_reference_reproduces_golden(seed):
    if not orc.ref_available():
        pytest.skip("oracle/_ref not built")
    script = (GOLD / f"store_script_{seed}.txt").read_text()
    assert orc.ref_store_script(script) == (GOLD / f"store_script_{seed}.expected").read_text()


def test_golden_scripts_cover_the_lifecycle():
    text = "".join((GOLD / f"store_script_{s}.expected").read_text() for s in SEEDS)
    script = "".join((GOLD / f"store_script_{s}.txt").read_text() for s in SEEDS)
    for op in ("insert", "setf", "setp", "poll", "complete", "purge_stale", "purge_inputs", "drop", "ready",
               "count", "release"):
        assert f"\n{op} " in "\n" + script or f"\n{op}\n" in "\n" + script, op
    for code in (5, 12, 13, 14, 17, 18, 26):  # the reference's error paths
        assert f"err {code}\n" in text, code
    assert "none\n" in text  # a poll with too few ready records returns nullopt


def test_rule_reward_and_advantages_kats():
    assert so.rule_reward([], [3, 1, 4]) == 0.0
    assert so.rule_reward([9, 3, 1, 4], [3, 1, 4]) == 1.0
    assert so.rule_reward([3, 1, 3, 1], [3, 1, 4]) == 2 / 3
    assert so.group_advantages([1.0, 1.0]) == [0.0, 0.0]  # all equal -> 0 (SPEC KAT)
