"""Host-side multi-process logic on CPU (gloo, world_size 2): the bench's
control-plane collectives and the agent-centric placement / token-balanced
row sharding used by DP gangs."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench
    d = bench.Dist()
    mx = d.max(float(rank + 1))
    sm = d.sum(float(rank + 1))
    ob = d.bcast_obj(b"x" * 128 if rank == 0 else None, src=0)
    d.barrier()
    d.close()
    q.put((rank, mx, sm, ob))


def test_gloo_control_plane_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = [q.get(timeout=120) for _ in ps]
    for p in ps:
        p.join(timeout=60)
    for rank, mx, sm, ob in out:
        assert mx == 2.0 and sm == 3.0 and ob == b"x" * 128


@pytest.mark.parametrize("world", [1, 2, 4, 8])
def test_placement(world):
    import bench
    agents = ["a0", "a1", "a2", "a3"]
    p = bench.placement(agents, world)
    if world >= 4:
        gangs = [tuple(v) for v in p.values()]
        assert all(len(g) == world // 4 for g in gangs)
        assert len(set(r for g in gangs for r in g)) == world  # disjoint, covering
    else:
        assert all(len(v) == 1 and 0 <= v[0] < world for v in p.values())


@pytest.mark.parametrize("M,g", [(16384, 2), (16384, 8), (1000, 3), (7, 4), (0, 2)])
def test_row_shards_partition(M, g):
    # the ranges fm_agent_set_shard trains: [M*r/g, M*(r+1)/g)
    spans = [(M * r // g, M * (r + 1) // g) for r in range(g)]
    assert spans[0][0] == 0 and spans[-1][1] == M
    assert all(spans[i][1] == spans[i + 1][0] for i in range(g - 1))
    assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1


def test_clock_sampler_window(tmp_path, monkeypatch):
    """bench.ClockSampler: start() waits for nvidia-smi's first sample, mark()
    opens the timed window, stop() keeps the window's samples (plus the first
    one after it) and reports the median SM clock and any throttle reasons —
    against a fake nvidia-smi printing a line every 50 ms."""
    import time
    import bench
    fake = tmp_path / "nvidia-smi"
    fake.write_text("#!/bin/sh\n"
                    "i=0\n"
                    "while true; do\n"
                    "  if [ $i -lt 3 ]; then r='Not Active'; else r='Active'; fi\n"
                    "  echo \"0, 1965, 1965, 700.0, 0x0, Not Active, Not Active, Not Active, $r\"\n"
                    "  i=$((i+1)); sleep 0.05\n"
                    "done\n")
    fake.chmod(0o755)
    monkeypatch.setenv("PATH", f"{tmp_path}:{os.environ['PATH']}")
    c = bench.ClockSampler(0)
    c.start()
    assert c.lines, "start() returns once the first sample arrived"
    time.sleep(0.3)  # warm-up steps
    c.mark()
    time.sleep(0.3)  # the timed region
    out = c.stop()
    assert out["sm_mhz"] == 1965.0 and out["sm_max_mhz"] == 1965.0
    assert 3 <= out["samples"] <= 10
    assert out["reasons"] == ["sw_power_cap"]
    assert c.proc.poll() is not None  # nvidia-smi stopped
