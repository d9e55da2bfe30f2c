"""Multi-process (world_size 2, gloo on CPU) coverage of the N>1 host logic:
frame sharding of a batch and the max-over-ranks timing reduction bench.py
uses.  No GPU needed."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

from paper_2305_02064_b200.shard import frame_range, max_over_ranks  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_frames, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lo, hi = frame_range(n_frames, rank, world)
    got = [None] * world
    dist.all_gather_object(got, (lo, hi))
    t = max_over_ranks(1.5 + rank, dist)
    if rank == 0:
        out.put((got, t))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("n_frames", [64, 7, 1])
def test_frame_sharding_gloo_world2(n_frames):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, n_frames, q)) for r in range(2)]
    for p in procs:
        p.start()
    ranges, tmax = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    # contiguous partition of [0, F), balanced to within one frame
    assert ranges[0][0] == 0 and ranges[-1][1] == n_frames
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(len(ranges) - 1))
    sizes = [h - lo for lo, h in ranges]
    assert max(sizes) - min(sizes) <= 1
    assert tmax == 2.5


def test_frame_range_single_and_errors():
    assert frame_range(5, 0, 1) == (0, 5)
    with pytest.raises(ValueError):
        frame_range(5, 2, 2)


def test_frame_subset_echo_matches_full_scene():
    """A rank's frames, synthesised on their own, are byte-identical to the
    same frames of the whole batch (noise counters shifted)."""
    import scenes
    sc = scenes.raster_scene(8, 6, 16, 16, 8, 8, 5e-3, 0.25, n_frames=3, jitter_xy=0.5e-3, jitter_z=1e-3, seed=3)
    rng = np.random.default_rng(0)
    pos = [np.array([[0.0, 0.0, 0.25]]) + rng.normal(0, 0.01, (2, 3)) for _ in range(3)]
    sc = scenes.dataclasses.replace(sc, scat_pos=pos, scat_amp=[np.ones(2, complex)] * 3)
    full = scenes.synthesize_cpu(sc)
    for lo, hi in ((0, 1), (1, 3), (2, 3)):
        sub = scenes.frame_subset(sc, lo, hi)
        assert np.array_equal(scenes.synthesize_cpu(sub), full[lo:hi])


# ---- slab decomposition: the exchange of sar_slab_stage's blocks ----------
def _xchg_worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2305_02064_b200.slab import exchange
    # block h of rank g holds 1000 g + 10 h + the element index
    send = torch.stack([torch.arange(6, dtype=torch.float32).reshape(2, 3) + 1000 * rank + 10 * h
                        for h in range(world)])
    recv = exchange(send)
    out.put((rank, send.numpy(), recv.numpy()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_slab_exchange_gloo(world):
    """exchange() (all_to_all_single, what NCCL runs on the GPUs) delivers
    block h of every rank g to rank h in order of g -- the layout
    sar_slab_stage expects -- and permute_blocks (the single-process
    emulation the GPU tests use) does the same permutation."""
    from paper_2305_02064_b200.slab import permute_blocks
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_xchg_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r, (s, rv)) for r, s, rv in (q.get(timeout=120) for _ in range(world)))
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    base = np.arange(6, dtype=np.float32).reshape(2, 3)
    emu = permute_blocks([torch.from_numpy(res[g][0]) for g in range(world)])
    for h in range(world):
        recv = res[h][1]
        for g in range(world):
            assert np.array_equal(recv[g], base + 1000 * g + 10 * h)
        assert np.array_equal(emu[h].numpy(), recv)
