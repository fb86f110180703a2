"""Synthetic experience sets shared by the golden-fixture generator and the tests.

C1: 2 agents, V=32, D=16, GRPO k=8, micro-batch 16, global 64,
policy-sampled EOS-terminated responses (policy.hpp:119-130 seeded as
rollout.hpp:638-645) rewarded by rule_reward(pattern {3,1,4})
(training.hpp:71-83, config.hpp:101) — generated with the compiled reference.
"mid": V=256, D=64 uniform tokens (the §8d recipe at a size the f64 oracle
finishes in milliseconds) — exercises the tensor-core path's tiling.
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as orc
from paper_2602_09578_b200 import workload as wl


def c1_samples(agent: str, n_updates: int = 2, max_tokens: int = 256, seed: int = 2048, V=32, D=16,
               G=64, k=8):
    """Returns (ids, turns, trajs, versions, samples[(prompt, resp)], rewards, advantages) in
    canonical order per version."""
    W0 = orc.seeded_weights(V, D, orc.agent_seed(seed, agent))
    ids, turns, trajs, versions, samples, rewards = [], [], [], [], [], []
    for u in range(n_updates):
        for i in range(G):
            qid = f"q{u * (G // k) + i // k:05d}"
            prompt = wl.query_prompt(seed, qid, V)
            sid = f"{qid}_0_{i % k}"
            tok_seed = wl.mix_u64(wl.mix_str(wl.mix_str(wl.mix_u64(seed, 0x70CE), agent), sid), u)
            resp, _ = orc.ref_generate(W0, prompt, max_tokens, tok_seed)
            ids.append(qid)
            turns.append(0)
            trajs.append(i % k)
            versions.append(u)
            samples.append((prompt.astype(np.int32), resp.astype(np.int32)))
            target = np.array([3, 1, 4], np.int32)  # kept alive across the C call
            rewards.append(orc.olib().fmo_rule_reward(resp.ctypes.data, len(resp), target.ctypes.data, 3))
    rewards = np.asarray(rewards)
    adv = np.concatenate([orc.group_advantages(rewards[g:g + k]) for g in range(0, len(rewards), k)])
    return ids, turns, trajs, versions, samples, rewards, adv


def uniform_samples(agent: str, V: int, n_updates: int, L: int, G=64, k=16, seed=2048):
    cfg = wl.Config("mid", (agent,), V, 64, group_k=k, global_batch=G, resp_len=L, seed=seed)
    ids, turns, trajs, versions, samples, rewards = [], [], [], [], [], []
    for u in range(n_updates):
        for s in wl.step_samples(cfg, agent, u):
            ids.append(s.input_id)
            turns.append(s.turns)
            trajs.append(s.traj)
            versions.append(u)
            samples.append((s.prompt, s.response))
            rewards.append(s.reward)
    rewards = np.asarray(rewards)
    adv = np.concatenate([orc.group_advantages(rewards[g:g + k]) for g in range(0, len(rewards), k)])
    return ids, turns, trajs, versions, samples, rewards, adv
