"""Agent-centric placement (host logic, CPU)."""
import pytest

from paper_2602_09578_b200.placement import agent_centric_plan, static_plan

AG = [f"agent{i}" for i in range(8)]


def c4_loads():  # 1 core agent with 76% of the micro-batches, 7 auxiliary agents
    l = {AG[0]: 6.0}
    l.update({a: 2.0 / 7 for a in AG[1:]})
    return l


@pytest.mark.parametrize("n,core,shared", [(8, 6, 2), (4, 3, 1), (2, 1, 1)])
def test_c4_agent_centric(n, core, shared):
    p = agent_centric_plan(c4_loads(), n)
    assert len(p.gangs["agent0"]) == core
    assert len(p.shared) == shared
    hosted = sorted(a for v in p.shared.values() for a in v)
    assert hosted == sorted(AG[1:])
    used = set(r for g in p.gangs.values() for r in g) | set(p.shared)
    assert used == set(range(n))
    assert not (set(r for g in p.gangs.values() for r in g) & set(p.shared))


def test_uniform_loads_one_gang_each():
    p = agent_centric_plan({a: 1.0 for a in AG[:4]}, 8)
    assert sorted(len(g) for g in p.gangs.values()) == [2, 2, 2, 2]
    assert not p.shared


def test_static_plan():
    p = static_plan(AG, 8)
    assert all(len(g) == 1 for g in p.gangs.values())
    p = static_plan(AG[:4], 2)
    assert p.shared == {0: ["agent0", "agent2"], 1: ["agent1", "agent3"]}


def test_drifting_core_moves_only_the_two_cores():
    """C4 with a drifting core (bench.py --c4-policy dynamic): between phases only
    the old and the new core change GPUs; every auxiliary agent keeps its GPU."""
    agents = [f"agent{i}" for i in range(8)]
    for n in (2, 4, 8):
        A = max(1, int(round(0.24 * n)))
        Cn = int(round(A * 0.76 / 0.24))

        def plan(core):
            return agent_centric_plan({a: (float(Cn) if a == core else A / 7) for a in agents}, n)

        def hosts(p, a):
            return p.gangs[a] if a in p.gangs else [r for r, v in p.shared.items() if a in v]

        p0, p1 = plan("agent0"), plan("agent1")
        moved = {a for a in agents if hosts(p0, a) != hosts(p1, a)}
        assert moved <= {"agent0", "agent1"}
        assert hosts(p1, "agent1") == hosts(p0, "agent0")  # the new core takes over the core gang
