"""Agent-centric placement of agents onto the GPUs of one box.

The reference binds each agent's process group gang-style to
`devices_per_group` free devices (STRICT_PACK, training.hpp:498-531) and
swaps idle agents out when training slots run short (orchestrator.hpp:387-416).
FlexMARL's point (§6) is that a skewed multi-agent workload should
not get one static slice per agent: GPUs follow the load.  This module turns
per-agent loads into a plan for one box:

  * agents whose load share warrants >= 1 GPU get a data-parallel gang of
    GPUs (largest-remainder apportionment of the box);
  * the remaining (auxiliary) agents are packed onto the leftover GPUs and
    time-multiplexed there with training-state swaps.

The plan is pure host logic (tested on CPU); bench.py executes it.
"""
from __future__ import annotations

from dataclasses import dataclass, field


@dataclass
class Plan:
    gangs: dict = field(default_factory=dict)     # agent -> list of ranks (DP gang, size >= 1)
    shared: dict = field(default_factory=dict)    # rank -> list of agents time-multiplexed on it

    def agents_on(self, rank: int) -> list:
        out = [a for a, g in self.gangs.items() if rank in g]
        return out + list(self.shared.get(rank, []))


def static_plan(agents: list, n_gpus: int) -> Plan:
    """One slice per agent (the baseline the paper argues against): agent i on
    GPU i mod N; with fewer GPUs than agents they share by round robin."""
    p = Plan()
    if n_gpus >= len(agents):
        for i, a in enumerate(agents):
            p.gangs[a] = [i]
        return p
    for i, a in enumerate(agents):
        p.shared.setdefault(i % n_gpus, []).append(a)
    return p


def agent_centric_plan(loads: dict, n_gpus: int, min_shared_gpus: int = 1) -> Plan:
    """loads: agent -> expected work (e.g. micro-batches per epoch).

    Agents with a share of at least one GPU get gangs sized by largest
    remainder; the others are packed (greedy, by load) onto the remaining
    GPUs, at least `min_shared_gpus` of which are reserved when such agents
    exist."""
    total = float(sum(loads.values()))
    if total <= 0 or n_gpus < 1:
        raise ValueError("need positive loads and at least one GPU")
    order = sorted(loads, key=lambda a: (-loads[a], a))
    big = [a for a in order if loads[a] / total * n_gpus >= 1.0]
    small = [a for a in order if a not in big]
    small_share = sum(loads[a] for a in small) / total * n_gpus
    reserve = min(n_gpus - 1, max(min_shared_gpus, int(round(small_share)))) if small else 0
    if not big:  # nobody earns a whole GPU: everything shares
        reserve = n_gpus
    avail = n_gpus - reserve
    p = Plan()
    if big:
        btotal = sum(loads[a] for a in big)
        quota = {a: loads[a] / btotal * avail for a in big}
        alloc = {a: max(1, int(quota[a])) for a in big}
        while sum(alloc.values()) > avail:  # more big agents than GPUs: demote the smallest
            a = min((x for x in alloc if alloc[x] == 1), key=lambda x: loads[x], default=None)
            if a is None:
                break
            del alloc[a]
            small.insert(0, a)
        rest = avail - sum(alloc.values())
        for a in sorted(alloc, key=lambda x: -(quota[x] - int(quota[x])))[:max(rest, 0)]:
            alloc[a] += 1
        r = 0
        for a in sorted(alloc, key=lambda x: -loads[x]):
            p.gangs[a] = list(range(r, r + alloc[a]))
            r += alloc[a]
        first_shared = r
    else:
        first_shared = 0
    shared_gpus = list(range(first_shared, n_gpus))
    if small:
        if not shared_gpus:
            raise ValueError("no GPU left for the auxiliary agents")
        load_on = {g: 0.0 for g in shared_gpus}
        for a in sorted(small, key=lambda x: (-loads[x], x)):
            g = min(shared_gpus, key=lambda x: (load_on[x], x))
            p.shared.setdefault(g, []).append(a)
            load_on[g] += loads[a]
    return p
