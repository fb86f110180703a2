"""Generates tests/golden/*.npz from the COMPILED REFERENCE (oracle/_ref).

Run in the CPU container (needs /root/reference to build oracle/_ref):
    python tests/golden/make_golden.py
Every array here comes out of the unmodified reference headers via
oracle/ref_driver.cpp; tests/test_oracle.py pins the C restatement against
them and the GPU tests compare the CUDA path with both.
"""
from __future__ import annotations

import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

from oracle import oracle as orc  # noqa: E402
import datasets  # noqa: E402

OUT = Path(__file__).resolve().parent


def _p(a):
    return a.ctypes.data


def gen_rng(L):
    seeds = np.array([0, 1, 2048, (1 << 63) + 5, 0xDEADBEEFCAFEBABE], dtype=np.uint64)
    out = {}
    for kind, name in ((0, "u64"), (1, "unit"), (2, "normal"), (3, "below")):
        rows = []
        for s in seeds:
            buf = np.zeros(64, dtype=np.uint64 if kind in (0, 3) else np.float64)
            L.ref_rng_draw(int(s), kind, 1000, 64, _p(buf))
            rows.append(buf)
        out[name] = np.stack(rows)
    out["seeds"] = seeds
    agents = ["planner", "executor", "critic", "agent0"]
    out["agent_names"] = np.array(agents)
    out["agent_seeds"] = np.array([L.ref_agent_seed(2048, a.encode()) for a in agents], dtype=np.uint64)
    out["mix_u64"] = np.array([L.ref_mix_u64(2048, 0x5EED), L.ref_mix_u64(7, 9)], dtype=np.uint64)
    out["mix_str"] = np.array([L.ref_mix_str(2048, b"q00001"), L.ref_mix_str(0, b"")], dtype=np.uint64)
    for a in ("planner", "executor"):
        w = np.zeros(32 * 16)
        L.ref_seeded_weights(32, 16, L.ref_agent_seed(2048, a.encode()), _p(w))
        out[f"W0_{a}"] = w.reshape(32, 16)
    np.savez_compressed(OUT / "rng.npz", **out)


def gen_adv_adam(L):
    rng = np.random.default_rng(7)
    groups = [np.array([1.0, 0, 1, 0]), np.full(8, 0.5), rng.random(16), np.array([3.0]),
              np.array([1e9, 1e9 + 1]), rng.normal(size=8) * 1e-12, np.array([0.0, 1.0, 0.0])]
    rewards = np.concatenate(groups)
    off = np.cumsum([0] + [len(g) for g in groups]).astype(np.int32)
    adv = np.zeros_like(rewards)
    for i, g in enumerate(groups):
        o = np.zeros(len(g))
        L.ref_group_advantages(_p(np.ascontiguousarray(g)), len(g), 1e-8, _p(o))
        adv[off[i]:off[i + 1]] = o
    # Adam: 3 steps over 64 params incl. the epsilon-sensitive regime
    n = 64
    w = rng.normal(size=n) * 0.5
    gs = [rng.normal(size=n) * 10.0 ** rng.integers(-12, -2, size=n) for _ in range(3)]
    gs[0][:4] = [1e-3, -1e-9, 0.0, 1e-8]
    ws, ms, vs = [], [], []
    W, M, Vv, st = w.copy(), np.zeros(n), np.zeros(n), np.zeros(1, dtype=np.int64)
    for g in gs:
        L.ref_adam_step(_p(W), _p(M), _p(Vv), _p(st), _p(np.ascontiguousarray(g)), n, 1e-6, 0.9, 0.999, 1e-8)
        ws.append(W.copy())
        ms.append(M.copy())
        vs.append(Vv.copy())
    np.savez_compressed(OUT / "adv_adam.npz", rewards=rewards, seg_off=off, adv=adv, w0=w, g=np.stack(gs),
                        w=np.stack(ws), m=np.stack(ms), v=np.stack(vs))


def gen_poll(L):
    rng = np.random.default_rng(11)
    n = 48
    ids = [f"q{int(x):05d}" for x in rng.integers(0, 12, size=n)]
    ids[3] = "q00003"
    ids[4] = "q10"      # non-numeric-width ids exercise lexicographic order
    ids[5] = "q1"
    turns = rng.integers(0, 3, size=n).astype(np.int32)
    trajs = rng.integers(0, 40, size=n).astype(np.int32)
    trajs[:] = np.arange(n)  # unique keys
    versions = rng.integers(0, 2, size=n).astype(np.int64)
    ready = (rng.random(n) > 0.2).astype(np.uint8)
    arr = (C.c_char_p * n)(*[s.encode() for s in ids])
    out = np.zeros(n, dtype=np.int32)
    got = L.ref_poll_order(n, arr, _p(turns), _p(trajs), _p(versions), _p(ready), 1, 5, _p(out))
    np.savez_compressed(OUT / "poll.npz", ids=np.array(ids), turns=turns, trajs=trajs, versions=versions,
                        ready=ready, current_version=1, mb=5, order=out[:got])


def _run_fixture(name, agent, V, D, data, n_updates, G=64, mb=16):
    ids, turns, trajs, versions, samples, rewards, adv = data
    order = np.random.default_rng(3).permutation(len(ids)).astype(np.int32)  # insertion != canonical
    r = orc.ref_run_agent(agent, V, D, 2048, G, mb, n_updates, ids, turns, trajs, versions, samples, adv,
                          insert_order=order)
    buf, poff, roff = orc.pack_payloads(samples)
    np.savez_compressed(OUT / f"{name}.npz", agent=agent, V=V, D=D, G=G, mb=mb, n_updates=n_updates,
                        ids=np.array(ids), turns=np.asarray(turns, np.int32), trajs=np.asarray(trajs, np.int32),
                        versions=np.asarray(versions, np.int64), payloads=buf, prompt_off=poff, resp_off=roff,
                        rewards=rewards, adv=adv, insert_order=order, poll_order=r["poll_order"], W0=r["W0"],
                        W=r["W"], m=r["m"], v=r["v"], mb_grad_norm=r["mb_grad_norm"],
                        upd_grad_norm=r["upd_grad_norm"])


def main():
    L = orc.rlib()
    gen_rng(L)
    gen_adv_adam(L)
    gen_poll(L)
    for agent in ("planner", "executor"):
        _run_fixture(f"c1_{agent}", agent, 32, 16, datasets.c1_samples(agent), 2)
    _run_fixture("mid_agent0", "agent0", 256, 64, datasets.uniform_samples("agent0", 256, 2, 48), 2)
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)


if __name__ == "__main__":
    main()
