"""Multi-process (N > 1) host logic of bench.py on CPU: world size 2 over gloo at 127.0.0.1.
The path shards as independent replicas: the only cross-rank step is the
aggregation of the timed region — max of the device time, sum of the iterations."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    import bench
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # replica r ran 13 + r iterations in 1.0 + 0.5 r seconds
        t, k = bench.aggregate_over_ranks(1.0 + 0.5 * rank, 13 + rank, world, "cpu")
        q.put((rank, t, k))
    finally:
        dist.destroy_process_group()


def test_aggregate_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    got = sorted(q.get(timeout=10) for _ in range(2))
    for rank, t, k in got:
        assert t == pytest.approx(1.5)       # slowest replica
        assert k == 27                       # all replicas' iterations
    # whole-job throughput: 27 iterations / 1.5 s
    assert got[0][2] / got[0][1] == pytest.approx(18.0)


def test_aggregate_single_rank_is_identity():
    import bench
    assert bench.aggregate_over_ranks(2.0, 5, 1, "cpu") == (2.0, 5)


def test_reference_arm_other_ranks_exit_silently():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                          "--steps", "1", "--warmup", "0"], env=env, capture_output=True, text=True, timeout=120)
    assert out.returncode == 0
    assert out.stdout.strip() == ""


@pytest.mark.gpu
def test_reference_arm_rank0_line():
    """The reference arm (the oracle on C4 n = 1024) takes the device-built setup: GPU box only."""
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "1", "--warmup", "0"], env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "iters/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
