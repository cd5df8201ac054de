"""Frame sharding logic with world_size 2 on the gloo backend (CPU)."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2010_08486_b200.sharding import ShardedRunner, gather_frame_results, owned_frames


def test_owned_frames_partition():
    for world in (1, 2, 3, 8):
        seen = []
        for r in range(world):
            seen += owned_frames(37, r, world)
        assert sorted(seen) == list(range(37))
    assert owned_frames(5, 1, 2) == [1, 3]
    with pytest.raises(ValueError):
        owned_frames(5, 2, 2)


def test_single_process_passthrough():
    out = ShardedRunner(lambda fr: [f.sum() for f in fr], 0, 1).run(
        lambda f: np.full((4, 4), f, np.float32), 5)
    assert out == [16.0 * f for f in range(5)]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_frames, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        calls = []

        def fake_detect(frames):          # CPU stand-in for Detector.run_batch
            calls.append(len(frames))
            return [np.array([(f.sum(), f.shape[0])], dtype=[("s", "f8"), ("n", "i4")]) for f in frames]

        runner = ShardedRunner(fake_detect)
        out = runner.run(lambda f: np.full((3, 3), f + 1, np.float32), n_frames)
        if rank == 0:
            q.put(("ok", [float(o["s"][0]) for o in out], calls))
        else:
            assert out is None
            q.put(("worker", rank, calls))
        # duplicated ownership must be detected on the gathering rank
        try:
            gather_frame_results({0: "x"}, 1)
            q.put(("dup", rank, "no error"))
        except RuntimeError as e:
            q.put(("dup", rank, str(e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_gather_in_frame_order():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    n_frames = 7
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_frames, q)) for r in range(2)]
    [p.start() for p in procs]
    msgs = [q.get(timeout=120) for _ in range(4)]
    [p.join(timeout=60) for p in procs]
    assert all(p.exitcode == 0 for p in procs)
    ok = [m for m in msgs if m[0] == "ok"][0]
    assert ok[1] == [9.0 * (f + 1) for f in range(n_frames)]
    assert ok[2] == [4]                                   # rank 0 owns frames 0, 2, 4, 6
    assert [m for m in msgs if m[0] == "worker"][0][2] == [3]
    dup = {m[1]: m[2] for m in msgs if m[0] == "dup"}
    assert "two ranks" in dup[0]
