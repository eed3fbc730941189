"""The N > 1 path of bench.py on CPU (world_size 2, gloo): one replica per rank, no data-path
collective, the job clock is the slowest rank (all_reduce MAX), throughput = ranks x units / time,
and the reference arm runs on rank 0 only."""
import os
import socket
import sys

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", init_method="env://", rank=rank, world_size=world)
    import bench
    r, w, _ = bench.dist_env()
    dist.barrier()
    ms = 10.0 + 5.0 * rank                       # rank 1 is the slow one
    mx = bench.max_over_ranks(ms, w, "cpu")
    rate = bench.job_rate(1000, 4, w, mx)
    out[rank] = (r, w, mx, rate)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_timing_and_rate():
    world, port = 2, _free_port()
    with mp.Manager() as mgr:
        out = mgr.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    for rank in range(world):
        r, w, mx, rate = res[rank]
        assert (r, w) == (rank, world)
        assert mx == 15.0                        # max over ranks, identical on every rank
        assert rate == pytest.approx(2 * 1000 * 4 / 15e-3)


def test_reference_arm_runs_on_rank_zero_only(capsys):
    import bench

    class Args:
        config, ref_angles, steps, warmup = 1, 2, 1, 0

    assert bench.reference_arm(Args, 1, 2) == 0
    assert capsys.readouterr().out == ""


def test_reference_arm_json_line(capsys):
    """--impl reference on rank 0: the fp64 oracle on a bounded sample, one JSON line."""
    import json

    import bench

    class Args:
        config, ref_angles, steps, warmup = 1, 2, 1, 0

    assert bench.reference_arm(Args, 0, 1) == 0
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "ray-samples/s" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "oracle" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["higher_is_better"] is True
