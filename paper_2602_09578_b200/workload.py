"""Synthetic experience for the benchmark configurations.

Host-side input generation only (never timed as part of the hot path):
  * splitmix64 streams restated from rng.hpp:14-64 (vectorised with numpy);
  * query ids ``q%05d`` and prompts as in workload.hpp:36-47
    (Rng(mix_u64(mix_str(mix_u64(seed, 0x9E77), input_id), 1)): length
    4 + next_below(5), tokens 1 + next_below(V - 1));
  * responses of fixed length L, i.i.d. next_below(V) from
    Rng(mix_u64(mix_str(mix_u64(seed, 0x5EED), agent), sample_idx));
  * rewards next_unit() from Rng(mix_u64(mix_str(mix_u64(seed, 0x5EEE), agent), sample_idx));
  * GRPO groups of k consecutive trajectories of one query.
The initial weights come from the native, bit-identical
``fm_seeded_weights`` (policy.hpp:29-35, training.hpp:245-248).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

M64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15


def splitmix64_draws(seed: int, n: int) -> np.ndarray:
    """The first n outputs of Rng(seed).next_u64() (rng.hpp:14-19, 40)."""
    with np.errstate(over="ignore"):
        i = np.arange(1, n + 1, dtype=np.uint64)
        z = np.uint64(seed & M64) + i * np.uint64(GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _splitmix_scalar(state: int) -> tuple[int, int]:
    state = (state + GOLDEN) & M64
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M64
    return state, z ^ (z >> 31)


def mix_u64(seed: int, value: int) -> int:  # rng.hpp:21-24
    s = (seed ^ ((value + GOLDEN + ((seed << 6) & M64) + (seed >> 2)) & M64)) & M64
    return _splitmix_scalar(s)[1]


def mix_str(seed: int, text: str) -> int:  # rng.hpp:26-34
    h = seed ^ 0xCBF29CE484222325
    for c in text.encode():
        h ^= c
        h = (h * 0x100000001B3) & M64
        h = mix_u64(h, c)
    return h


def next_unit(seed: int, n: int) -> np.ndarray:  # rng.hpp:43-48
    u = (splitmix64_draws(seed, n) >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
    return np.where(u <= 0.0, 2.0 ** -53, u)


def encode_tokens(tokens: np.ndarray) -> bytes:  # codec.hpp:15-22
    t = np.asarray(tokens, dtype=np.int64).astype("<u8")
    return np.uint64(len(t)).astype("<u8").tobytes() + t.tobytes()


def decode_tokens(payload: bytes) -> np.ndarray:  # codec.hpp:24-30
    n = int(np.frombuffer(payload[:8], dtype="<u8")[0])
    return np.frombuffer(payload[8:8 + 8 * n], dtype="<u8").astype(np.uint32).view(np.int32).copy()


def query_prompt(seed: int, input_id: str, vocab: int) -> np.ndarray:  # workload.hpp:36-47
    st = mix_u64(mix_str(mix_u64(seed, 0x9E77), input_id), 1)
    d = splitmix64_draws(st, 9)
    length = 4 + int(d[0] % np.uint64(5))
    return (1 + d[1:1 + length] % np.uint64(vocab - 1)).astype(np.int32)


@dataclass(frozen=True)
class Config:
    name: str
    agents: tuple[str, ...]
    vocab: int
    feat: int
    group_k: int = 16
    micro_batch: int = 16
    global_batch: int = 64
    resp_len: int = 1024
    seed: int = 2048
    lr: float = 1e-6

    @property
    def params(self) -> int:
        return self.vocab * self.feat

    @property
    def flops_per_token(self) -> int:  # 4*V*D (2VD logits + 2VD weight gradient)
        return 4 * self.vocab * self.feat


# BASELINE.json configs; C2 is the N=1 bench workload.
CONFIGS = {
    "C1": Config("C1", ("planner", "executor"), 32, 16, group_k=8, resp_len=32),
    "C2": Config("C2", ("agent0", "agent1", "agent2", "agent3"), 32000, 4096),
    "C3": Config("C3", ("agent0", "agent1", "agent2", "agent3"), 32000, 32768),
    "C4": Config("C4", tuple(f"agent{i}" for i in range(8)), 32000, 4096),
    "C5": Config("C5", ("agent0",), 128000, 8192, resp_len=4096),
}


@dataclass
class Sample:
    input_id: str
    turns: int
    traj: int
    prompt: np.ndarray
    response: np.ndarray
    reward: float
    advantage: float = 0.0
    prompt_payload: bytes = field(default=b"", repr=False)
    response_payload: bytes = field(default=b"", repr=False)


def step_samples(cfg: Config, agent: str, step: int, n: int | None = None,
                 resp_len: int | None = None) -> list[Sample]:
    """The global batch of `agent` at `step` (G samples in G/k GRPO groups),
    or its first n samples.  Advantages are NOT filled here: the caller runs
    the device K-adv kernel (fm_group_advantages) or the oracle."""
    G, k = cfg.global_batch, cfg.group_k
    L = cfg.resp_len if resp_len is None else resp_len
    n = G if n is None else n
    seed_tok = mix_str(mix_u64(cfg.seed, 0x5EED), agent)
    seed_rew = mix_str(mix_u64(cfg.seed, 0x5EEE), agent)
    out = []
    for i in range(n):
        sidx = step * G + i
        qid = f"q{step * (G // k) + i // k:05d}"
        prompt = query_prompt(cfg.seed, qid, cfg.vocab)
        resp = (splitmix64_draws(mix_u64(seed_tok, sidx), L) % np.uint64(cfg.vocab)).astype(np.int32)
        reward = float(next_unit(mix_u64(seed_rew, sidx), 1)[0])
        s = Sample(qid, 0, i % k, prompt, resp, reward)
        s.prompt_payload = encode_tokens(prompt)
        s.response_payload = encode_tokens(resp)
        out.append(s)
    return out


def group_offsets(samples: list[Sample]) -> np.ndarray:
    """Segment offsets of consecutive samples sharing an input_id."""
    off = [0]
    for i in range(1, len(samples)):
        if samples[i].input_id != samples[i - 1].input_id:
            off.append(i)
    off.append(len(samples))
    return np.asarray(off, dtype=np.int32)
