"""N > 1 plumbing of bench.py on CPU (gloo, world size 2).

The path does not shard (replicas only), so the multi-GPU
contract is: every rank runs its own replica, the timed region is bracketed
by barriers, `value` = total V-cycles over all ranks / max-over-ranks time,
and only rank 0 prints.  These tests exercise exactly that host logic
(bench.dist_env, bench.reduce_max_sum, the rank gating of the reference arm)
with two gloo processes on 127.0.0.1.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank),
                      MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r, w, lr = bench.dist_env()
    # rank r "timed" 1.0 + r seconds and ran 5 + r cycles
    t_max, c_sum = bench.reduce_max_sum(1.0 + r, 5 + r, "cpu")
    dist.barrier()
    dist.destroy_process_group()
    q.put((r, w, lr, t_max, c_sum))


def test_reduce_max_sum_gloo_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    out = sorted(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    assert [o[:3] for o in out] == [(0, 2, 0), (1, 2, 1)]
    for o in out:
        assert o[3] == 2.0          # max over ranks of the device time
        assert o[4] == 11.0         # sum over ranks of the cycles: value = 11 / 2.0


def test_reduce_is_identity_without_process_group():
    sys.path.insert(0, ROOT)
    import bench
    assert bench.reduce_max_sum(3.5, 7, "cpu") == (3.5, 7.0)


def test_reference_arm_under_torchrun_world2():
    """`bench.py --impl reference` launched like the driver does (torchrun,
    2 ranks): rank 0 alone runs the oracle and prints ONE JSON line; the other
    rank exits 0 without work."""
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--impl", "reference", "--gpus", "2", "--config", "1", "--steps", "1", "--warmup", "0"]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    res = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    lines = [l for l in res.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, res.stdout
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] == 1
