"""The source-level drop-in (dropin/marlsim/training.hpp) driven by the
reference's own Orchestrator (orchestrator.hpp, unmodified), against the
stock reference build of the same driver (SURVEY.md §4 test tier 4).

oracle/Makefile's `orch` target compiles tests/orch_driver.cpp twice in the
CPU container (the reference headers are there): oracle/_ref/orch_stock and
oracle/_ref/orch_b200 (-I dropin before the reference's include dir, linked to
libflexmarl_b200.so).  Both travel to the GPU box with the repo snapshot.

The drop-in keeps the reference's virtual-time bookkeeping, object-store
traffic and checkpoint byte lengths, so the two runs must produce the same
event sequence — every activate / suspend / micro_grad / update record with
the same virtual timestamp, agent, versions, sample counts and checkpoint
sizes — and only the arithmetic differs: grad norms and final weights within
the precision's contract (PARITY_F64 ~1e-9; BF16_TC the §8c contract).

Configs: the default RunConfig (3 agents, C1 dims V=32 D=16, GRPO k=16,
micro-batch 16 / global 64) with static allocation (no swaps; the reference's
PolicyState::deserialize transposes W when V != D, training.hpp:146), and with
2 training slots at V = D = 16, where the orchestrator suspends and re-activates
agents mid-step (checkpoints through the GPU's PolicyState serialisation).
"""
import json
import os
import subprocess
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
STOCK = ROOT / "oracle" / "_ref" / "orch_stock"
B200 = ROOT / "oracle" / "_ref" / "orch_b200"

CASES = [
    pytest.param(["2", "1", "2"], id="static-allocation"),
    pytest.param(["3", "0", "2", "16", "16"], id="swaps-midstep"),
]


def _run(binary, out, args, precision=None):
    out.mkdir(parents=True, exist_ok=True)
    env = dict(os.environ)
    if precision:
        env["FLEXMARL_PRECISION"] = precision
    r = subprocess.run([str(binary), str(out), *args], capture_output=True, text=True, env=env, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    events = [json.loads(l) for l in (out / "events.ndjson").read_text().splitlines()]
    agents = sorted({e["agent"] for e in events})
    w = {a: (np.fromfile(out / f"{a}.w0"), np.fromfile(out / f"{a}.w")) for a in agents}
    return events, w


@pytest.mark.parametrize("args", CASES)
@pytest.mark.parametrize("precision", ["f64", "bf16"])
def test_reference_orchestrator_drives_b200_trainer(tmp_path, args, precision):
    if not (STOCK.exists() and B200.exists()):
        pytest.skip("drop-in harness not built (oracle/Makefile orch; needs the reference headers)")
    ev_ref, w_ref = _run(STOCK, tmp_path / "stock", args)
    ev, w = _run(B200, tmp_path / "b200", args, precision)
    assert len(ev) == len(ev_ref) and len(ev_ref) > 0
    kinds = [e["kind"] for e in ev_ref]
    assert kinds.count("micro_grad") >= 24 and kinds.count("update") >= 6
    if args[1] == "0":
        assert kinds.count("suspend") > 0
    tol = 1e-9 if precision == "f64" else 2e-2
    for a, b in zip(ev, ev_ref):
        assert a["kind"] == b["kind"] and a["agent"] == b["agent"] and a["t"] == b["t"], (a, b)
        for k in b:
            if k == "grad_norm":
                assert abs(a[k] - b[k]) <= tol * abs(b[k]), (a, b)
            else:
                assert a[k] == b[k], (k, a, b)
    n_upd = {}
    for e in ev_ref:
        if e["kind"] == "update":
            n_upd[e["agent"]] = e["version"]
    for agent, (w0_ref, wf_ref) in w_ref.items():
        w0, wf = w[agent]
        assert np.array_equal(w0, w0_ref)  # PolicyModel::seeded, bit-exact
        d, d_ref = wf - w0, wf_ref - w0_ref
        rel = float(np.linalg.norm(d - d_ref) / np.linalg.norm(d_ref))
        off = float(np.mean(np.abs(d - d_ref) > 0.5 * 1e-6 * n_upd[agent]))
        print(f"{precision} {args} {agent}: delta-W rel-Fro {rel:.3e}, elements off {off:.2e}")
        if precision == "f64":
            assert rel <= 1e-6
        else:
            assert rel <= 5e-2 and off <= 1e-2
