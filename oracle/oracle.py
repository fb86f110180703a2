"""oracle/oracle.py — TEST INFRASTRUCTURE ONLY (the parity checker).

numpy/ctypes front end of
  * ``oracle/libflexmarl_oracle.so`` — our plain-C restatement of the
    reference path (oracle/flexmarl_oracle.c, every function cites the
    reference file:line it restates), and
  * ``oracle/_ref/libmarlsim_ref.so`` — the UNMODIFIED reference headers
    compiled with a thin extern "C" driver (oracle/ref_driver.cpp).

The restatement is pinned against the reference by tests/test_oracle.py
(golden fixtures in tests/golden/ generated from _ref by
tests/golden/make_golden.py, plus live cross-checks when _ref is built).
Only tests/, __graft_entry__.smoke() and bench.py's reference /
cpu_baseline legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ORACLE_SO = HERE / "libflexmarl_oracle.so"
REF_SO = HERE / "_ref" / "libmarlsim_ref.so"
REF_INC = Path("/root/reference/proj/include")

P = C.c_void_p
U64, I64, I, D = C.c_uint64, C.c_int64, C.c_int, C.c_double


def build(ref: bool = True) -> None:
    """Builds the restatement, and _ref when the reference sources exist."""
    targets = ["liboracle"]
    if ref and REF_INC.exists():
        targets += ["ref", "orch"]  # orch: the drop-in harness (needs the native library, built first)
    subprocess.run(["make", "-s", "-C", str(HERE), *targets], check=True)


_o = None
_r = None


def olib() -> C.CDLL:
    global _o
    if _o is None:
        if not ORACLE_SO.exists():
            build(ref=False)
        L = C.CDLL(str(ORACLE_SO))
        L.fmo_mix_u64.restype = U64
        L.fmo_mix_u64.argtypes = [U64, U64]
        L.fmo_mix_str.restype = U64
        L.fmo_mix_str.argtypes = [U64, C.c_char_p]
        L.fmo_agent_seed.restype = U64
        L.fmo_agent_seed.argtypes = [U64, C.c_char_p]
        L.fmo_rng_draw.argtypes = [U64, I, U64, U64, P]
        L.fmo_seeded_weights.argtypes = [U64, U64, U64, P]
        L.fmo_group_advantages.argtypes = [P, I, D, P]
        L.fmo_rule_reward.restype = D
        L.fmo_rule_reward.argtypes = [P, I, P, I]
        L.fmo_adam_step.argtypes = [P, P, P, P, P, U64, D, D, D, D]
        L.fmo_decode_tokens.restype = U64
        L.fmo_decode_tokens.argtypes = [P, P]
        L.fmo_encode_tokens.restype = U64
        L.fmo_encode_tokens.argtypes = [P, U64, P]
        L.fmo_featurize.argtypes = [U64, U64, P, I, P]
        L.fmo_probabilities.argtypes = [U64, U64, P, P, I, P]
        L.fmo_log_prob.restype = D
        L.fmo_log_prob.argtypes = [U64, U64, P, P, I, I]
        L.fmo_accumulate_grad.argtypes = [U64, U64, P, P, I, I, D, P]
        L.fmo_poll_select.restype = I
        L.fmo_poll_select.argtypes = [I, P, P, P, P, P, P, I64, I64, P]
        L.fmo_pack_rows.restype = I64
        L.fmo_pack_rows.argtypes = [I, P, P, P, P, I64, P, P, P, P, P]
        L.fmo_run_agent.restype = I
        L.fmo_run_agent.argtypes = [U64, U64, I64, I64, I, P, P, P, P, D, D, D, D, P, P, P, P, P, P, P]
        L.fmo_sparse_grad.restype = I64
        L.fmo_sparse_grad.argtypes = [U64, U64, U64, I, P, P, P, P, I64, I64, P, P, P]
        L.fmo_step_grad.restype = I
        L.fmo_step_grad.argtypes = [U64, U64, P, I, P, P, P, P, I64, I, I, P, P]
        _o = L
    return _o


def ref_available() -> bool:
    return REF_SO.exists()


def rlib() -> C.CDLL:
    global _r
    if _r is None:
        if not REF_SO.exists():
            if REF_INC.exists():
                build(ref=True)
            else:
                raise FileNotFoundError(f"{REF_SO} not built and reference sources absent")
        L = C.CDLL(str(REF_SO))
        L.ref_last_error.restype = C.c_char_p
        L.ref_agent_seed.restype = U64
        L.ref_agent_seed.argtypes = [U64, C.c_char_p]
        L.ref_mix_u64.restype = U64
        L.ref_mix_u64.argtypes = [U64, U64]
        L.ref_mix_str.restype = U64
        L.ref_mix_str.argtypes = [U64, C.c_char_p]
        L.ref_rng_draw.argtypes = [U64, I, U64, U64, P]
        L.ref_seeded_weights.argtypes = [U64, U64, U64, P]
        L.ref_group_advantages.argtypes = [P, I, D, P]
        L.ref_rule_reward.restype = D
        L.ref_rule_reward.argtypes = [P, I, P, I]
        L.ref_adam_step.argtypes = [P, P, P, P, P, U64, D, D, D, D]
        L.ref_featurize.argtypes = [U64, U64, P, I, P]
        L.ref_probabilities.argtypes = [U64, U64, P, P, I, P]
        L.ref_accumulate_grad.argtypes = [U64, U64, P, P, I, I, D, P]
        L.ref_generate.restype = I
        L.ref_generate.argtypes = [U64, U64, P, P, I, I, U64, P, P]
        L.ref_run_agent.restype = I
        L.ref_run_agent.argtypes = [C.c_char_p, U64, U64, U64, I64, I64, I, I, P, P, P, P, P, P, P, P, P, D,
                                    P, P, P, P, P, P, P, P, P, I]
        L.ref_serialize_state.restype = U64
        L.ref_serialize_state.argtypes = [I64, I64, I64, U64, U64, P, P, P, P, U64]
        L.ref_deserialize_state.restype = I
        L.ref_deserialize_state.argtypes = [P, U64, P, P, P, P, P]
        L.ref_poll_order.restype = I
        L.ref_poll_order.argtypes = [I, P, P, P, P, P, I64, I64, P]
        L.ref_store_script.restype = U64
        L.ref_store_script.argtypes = [C.c_char_p, C.c_char_p, U64]
        _r = L
    return _r


def _p(a: np.ndarray) -> int:
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data


# ---------------------------------------------------------------------------
# payload packing shared by the restatement and the reference driver
# ---------------------------------------------------------------------------
def encode(tokens) -> bytes:
    t = np.asarray(tokens, dtype=np.int64).astype("<u8")
    return np.uint64(len(t)).astype("<u8").tobytes() + t.tobytes()


def pack_payloads(samples) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
    """samples: iterable of (prompt_tokens, response_tokens) -> buffer, prompt_off, resp_off."""
    chunks, poff, roff, pos = [], [], [], 0
    for prompt, resp in samples:
        for arr, offs in ((prompt, poff), (resp, roff)):
            b = encode(arr)
            offs.append(pos)
            chunks.append(b)
            pos += len(b)
    buf = np.frombuffer(b"".join(chunks) or b"\0", dtype=np.uint8).copy()
    return buf, np.asarray(poff, dtype=np.int64), np.asarray(roff, dtype=np.int64)


# ---------------------------------------------------------------------------
# restatement wrappers
# ---------------------------------------------------------------------------
def seeded_weights(V, D_, seed) -> np.ndarray:
    w = np.empty(V * D_, dtype=np.float64)
    olib().fmo_seeded_weights(V, D_, seed, _p(w))
    return w.reshape(V, D_)


def agent_seed(seed, agent) -> int:
    return olib().fmo_agent_seed(seed, agent.encode())


def group_advantages(rewards, eps=1e-8) -> np.ndarray:
    r = np.ascontiguousarray(rewards, dtype=np.float64)
    out = np.zeros_like(r)
    olib().fmo_group_advantages(_p(r), len(r), eps, _p(out))
    return out


def adam_step(w, m, v, step, g, lr=1e-6, b1=0.9, b2=0.999, eps=1e-8):
    w, m, v = (np.ascontiguousarray(x, dtype=np.float64).copy() for x in (w, m, v))
    g = np.ascontiguousarray(g, dtype=np.float64)
    st = np.array([step], dtype=np.int64)
    olib().fmo_adam_step(_p(w), _p(m), _p(v), _p(st), _p(g), w.size, lr, b1, b2, eps)
    return w, m, v, int(st[0])


def probabilities(W, ctx) -> np.ndarray:
    W = np.ascontiguousarray(W, dtype=np.float64)
    c = np.ascontiguousarray(ctx, dtype=np.int32)
    out = np.empty(W.shape[0], dtype=np.float64)
    olib().fmo_probabilities(W.shape[0], W.shape[1], _p(W), _p(c), len(c), _p(out))
    return out


def poll_select(ids, turns, trajs, versions, ready, processing, current_version, mb) -> list:
    n = len(ids)
    arr = (C.c_char_p * max(n, 1))(*[s.encode() for s in ids])
    t = np.ascontiguousarray(turns, dtype=np.int32)
    j = np.ascontiguousarray(trajs, dtype=np.int32)
    v = np.ascontiguousarray(versions, dtype=np.int64)
    r = np.ascontiguousarray(ready, dtype=np.uint8)
    p = np.ascontiguousarray(processing, dtype=np.uint8)
    out = np.zeros(max(mb, 1), dtype=np.int32)
    got = olib().fmo_poll_select(n, arr, _p(t), _p(j), _p(v), _p(r), _p(p), current_version, mb, _p(out))
    return [] if got <= 0 else out[:got].tolist()


def pack_rows(samples, advantages, G) -> dict:
    """The bit-exact target of the device gather (fmo_pack_rows)."""
    buf, poff, roff = pack_payloads(samples)
    adv = np.ascontiguousarray(advantages, dtype=np.float64)
    M = int(sum(len(r) for _, r in samples))
    out = dict(action=np.zeros(M, np.int32), ctx4=np.zeros((M, 4), np.int32), n_ctx=np.zeros(M, np.int32),
               sample=np.zeros(M, np.int32), coef=np.zeros(M, np.float32))
    got = olib().fmo_pack_rows(len(samples), _p(buf), _p(poff), _p(roff), _p(adv), G, _p(out["action"]),
                               _p(out["ctx4"]), _p(out["n_ctx"]), _p(out["sample"]), _p(out["coef"]))
    assert got == M
    return out


def run_agent(V, D_, G, mb, n_updates, samples, advantages, W0, lr=1e-6, b1=0.9, b2=0.999, eps=1e-8,
              want_logp=False) -> dict:
    """samples/advantages in poll (canonical) order, G per update."""
    buf, poff, roff = pack_payloads(samples)
    adv = np.ascontiguousarray(advantages, dtype=np.float64)
    W = np.ascontiguousarray(W0, dtype=np.float64).reshape(-1).copy()
    m = np.zeros_like(W)
    v = np.zeros_like(W)
    mbn = np.zeros(n_updates * (G // mb), dtype=np.float64)
    upd = np.zeros(n_updates, dtype=np.float64)
    ntok = int(sum(len(r) for _, r in samples))
    logp = np.zeros(max(ntok, 1), dtype=np.float64) if want_logp else None
    last = np.zeros_like(W)
    olib().fmo_run_agent(V, D_, G, mb, n_updates, _p(buf), _p(poff), _p(roff), _p(adv), lr, b1, b2, eps,
                         _p(W), _p(m), _p(v), _p(mbn), _p(upd), _p(logp) if want_logp else None, _p(last))
    return dict(W=W.reshape(V, D_), m=m.reshape(V, D_), v=v.reshape(V, D_), mb_grad_norm=mbn,
                upd_grad_norm=upd, logp=logp[:ntok] if want_logp else None, last_grad=last.reshape(V, D_))


def sparse_grad(V, D_, seed, samples, advantages, G, max_cols=4096) -> dict:
    """First-update gradient -(1/G) sum_s A_s term_s of a few samples at full
    V x D, on the feature columns their contexts touch (fmo_sparse_grad:
    bit-identical to run_agent's last_grad there, every other column 0) and the
    micro-batch grad norm (training.hpp:417).  W comes from the seeded stream."""
    buf, poff, roff = pack_payloads(samples)
    adv = np.ascontiguousarray(advantages, dtype=np.float64)
    cols = np.zeros(max_cols, dtype=np.int64)
    grad = np.zeros(V * max_cols, dtype=np.float64)
    mbn = np.zeros(1, dtype=np.float64)
    nc = olib().fmo_sparse_grad(V, D_, seed, len(samples), _p(buf), _p(poff), _p(roff), _p(adv), G, max_cols,
                                _p(cols), _p(grad), _p(mbn))
    assert nc >= 0, "too many feature columns"
    return dict(cols=cols[:nc].copy(), grad=grad[:V * nc].reshape(V, nc).copy(), mb_grad_norm=float(mbn[0]))


def step_grad(V, D_, Wt, samples, advantages, G, mb=16, threads=0, mb_norms=True) -> dict:
    """Full-size gradient of one global step (fmo_step_grad): gradT [D][V]
    = -(1/G) sum_s A_s term_s, bit-identical to run_agent's dense arithmetic,
    and the per-micro-batch grad norms.  Wt = W transposed [D][V] f64."""
    import os
    buf, poff, roff = pack_payloads(samples)
    adv = np.ascontiguousarray(advantages, dtype=np.float64)
    Wt = np.ascontiguousarray(Wt, dtype=np.float64)
    gradT = np.empty((D_, V), dtype=np.float64)
    nmb = (len(samples) + mb - 1) // mb
    norms = np.zeros(nmb) if mb_norms else None
    th = threads or max(1, min(64, os.cpu_count() or 1))
    rc = olib().fmo_step_grad(V, D_, _p(Wt), len(samples), _p(buf), _p(poff), _p(roff), _p(adv), G, mb, th,
                              _p(gradT), _p(norms) if mb_norms else None)
    assert rc == 0, "fmo_step_grad: allocation failed"
    return dict(gradT=gradT, mb_grad_norms=norms)


# ---------------------------------------------------------------------------
# reference (compiled, unmodified headers) wrappers
# ---------------------------------------------------------------------------
def ref_run_agent(agent, V, D_, seed, G, mb, n_updates, ids, turns, trajs, versions, samples, advantages,
                  insert_order=None, lr=1e-6, want_state=True, skip_update=False) -> dict:
    L = rlib()
    n = len(ids)
    arr = (C.c_char_p * n)(*[s.encode() for s in ids])
    t = np.ascontiguousarray(turns, dtype=np.int32)
    j = np.ascontiguousarray(trajs, dtype=np.int32)
    ver = np.ascontiguousarray(versions, dtype=np.int64)
    buf, poff, roff = pack_payloads(samples)
    adv = np.ascontiguousarray(advantages, dtype=np.float64)
    order = np.arange(n, dtype=np.int32) if insert_order is None else np.ascontiguousarray(insert_order, np.int32)
    P_ = V * D_
    W0 = np.zeros(P_)
    W = np.zeros(P_)
    m = np.zeros(P_)
    v = np.zeros(P_)
    polled = np.zeros(n, dtype=np.int32)
    mbn = np.zeros(n_updates * (G // mb))
    upd = np.zeros(n_updates)
    tt = np.zeros(1)
    tu = np.zeros(1)
    rc = L.ref_run_agent(agent.encode(), V, D_, seed, G, mb, n_updates, n, arr, _p(t), _p(j), _p(ver), _p(buf),
                         _p(poff), _p(roff), _p(adv), _p(order), lr,
                         _p(W0) if want_state else None, _p(W) if want_state else None,
                         _p(m) if want_state else None, _p(v) if want_state else None,
                         _p(polled), _p(mbn), _p(upd), _p(tt), _p(tu), int(skip_update))
    if rc != 0:
        raise RuntimeError(f"ref_run_agent failed ({rc}): {L.ref_last_error().decode()}")
    return dict(W0=W0.reshape(V, D_), W=W.reshape(V, D_), m=m.reshape(V, D_), v=v.reshape(V, D_),
                poll_order=polled, mb_grad_norm=mbn, upd_grad_norm=upd, t_train=float(tt[0]),
                t_update=float(tu[0]))


def ref_generate(W, prompt, max_tokens, tok_seed):
    W = np.ascontiguousarray(W, dtype=np.float64)
    p = np.ascontiguousarray(prompt, dtype=np.int32)
    toks = np.zeros(max_tokens, dtype=np.int32)
    lps = np.zeros(max_tokens, dtype=np.float64)
    n = rlib().ref_generate(W.shape[0], W.shape[1], _p(W), _p(p), len(p), max_tokens, tok_seed, _p(toks), _p(lps))
    return toks[:n].copy(), lps[:n].copy()


def ref_serialize_state(version, step, samples, W, m, v) -> bytes:
    W = np.ascontiguousarray(W, dtype=np.float64)
    V, D_ = W.shape
    m = None if m is None else np.ascontiguousarray(m, dtype=np.float64)
    v = None if v is None else np.ascontiguousarray(v, dtype=np.float64)
    L = rlib()
    n = L.ref_serialize_state(version, step, samples, V, D_, _p(W), _p(m) if m is not None else None,
                              _p(v) if v is not None else None, None, 0)
    out = np.zeros(n, dtype=np.uint8)
    L.ref_serialize_state(version, step, samples, V, D_, _p(W), _p(m) if m is not None else None,
                          _p(v) if v is not None else None, _p(out), n)
    return out.tobytes()


def ref_deserialize_state(blob: bytes, P_: int) -> dict:
    buf = np.frombuffer(blob, dtype=np.uint8).copy()
    r, c, ver, cn = (np.zeros(1, np.uint64), np.zeros(1, np.uint64), np.zeros(1, np.int64), np.zeros(1, np.uint64))
    W = np.zeros(P_)
    rc = rlib().ref_deserialize_state(_p(buf), len(buf), _p(r), _p(c), _p(W), _p(ver), _p(cn))
    if rc != 0:
        raise RuntimeError(rlib().ref_last_error().decode())
    return dict(rows=int(r[0]), cols=int(c[0]), W=W, version=int(ver[0]), cache_n=int(cn[0]))


def ref_store_script(script: str) -> str:
    """Replays a store lifecycle script on the reference ExperienceStore (oracle/_ref)."""
    L = rlib()
    n = L.ref_store_script(script.encode(), None, 0)
    if n == 0:
        raise RuntimeError(L.ref_last_error().decode())
    buf = C.create_string_buffer(int(n))
    L.ref_store_script(script.encode(), buf, n)
    return buf.value.decode()
