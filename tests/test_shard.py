"""Multi-GPU partitioning logic, exercised on CPU: stripe planning and a
world_size-2 gloo run where each rank filters its stripe (with the oracle
standing in for the device filter) and rank 0 checks the stitched result."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2505_22938_b200 import FilterParams, ShapeSpec
from paper_2505_22938_b200.shard import assemble, filter_stripe, image_shard, stripe_plan


def _oracle_fn(img, params):
    return oracle.fast_filter(img, params.shape, params.percentile, params.boundary, threads=2)


@pytest.mark.parametrize("boundary", ["replicate", "valid"])
@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_stripes_stitch_to_whole_image(boundary, world):
    rng = np.random.default_rng(world)
    img = rng.integers(0, 65536, (37, 29, 3)).astype(np.uint16)
    params = FilterParams(shape=ShapeSpec("circle", 4), boundary=boundary)
    plan = stripe_plan(img.shape[0], 4, boundary, world)
    assert sum(s.rows for s in plan) == (img.shape[0] - 8 if boundary == "valid" else img.shape[0])
    parts = [filter_stripe(img, params, s, _oracle_fn) for s in plan]
    whole = _oracle_fn(img, params)
    assert np.array_equal(assemble(plan, parts), whole)


def test_image_shard_round_robin():
    got = [image_shard(64, 8, r) for r in range(8)]
    assert sorted(i for g in got for i in g) == list(range(64))
    assert all(len(g) == 8 for g in got)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, img, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    params = FilterParams(shape=ShapeSpec("circle", 6))
    plan = stripe_plan(img.shape[0], 6, "replicate", world)
    part = filter_stripe(img, params, plan[rank], _oracle_fn)
    parts = [None] * world
    dist.all_gather_object(parts, part)
    if rank == 0:
        q.put(assemble(plan, parts))
    dist.destroy_process_group()


def test_gloo_world2_stripes():
    img = np.random.default_rng(5).integers(0, 256, (61, 47)).astype(np.uint8)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, img, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert np.array_equal(out, _oracle_fn(img, FilterParams(shape=ShapeSpec("circle", 6))))


@pytest.mark.parametrize("boundary", ["replicate", "valid"])
def test_stripes_with_percentile_map(boundary):
    """A per-pixel percentile map of the FULL output shape (SPEC Fig. 12) is
    sliced to each stripe's rows (tiling.py:165-177 map -> targets)."""
    rng = np.random.default_rng(17)
    img = rng.integers(0, 256, (45, 31)).astype(np.uint8)
    r = 3
    oh = 45 - 2 * r if boundary == "valid" else 45
    ow = 31 - 2 * r if boundary == "valid" else 31
    pmap = rng.random((oh, ow))
    params = FilterParams(shape=ShapeSpec("circle", r), percentile=pmap, boundary=boundary)
    plan = stripe_plan(img.shape[0], r, boundary, 3)
    parts = [filter_stripe(img, params, s, _oracle_fn) for s in plan]
    assert np.array_equal(assemble(plan, parts), _oracle_fn(img, params))


def _gpu_worker(rank, world, port, img, q):
    """One rank of a gloo job filtering its stripe with the CUDA engine."""
    import torch
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(rank % torch.cuda.device_count())
    params = FilterParams(shape=ShapeSpec("circle", 7))
    plan = stripe_plan(img.shape[0], 7, "replicate", world)
    part = filter_stripe(img, params, plan[rank])  # default: the GPU filter_image
    parts = [None] * world
    dist.all_gather_object(parts, part)
    if rank == 0:
        q.put(assemble(plan, parts))
    dist.destroy_process_group()


@pytest.mark.gpu
def test_gloo_world2_gpu_stripes():
    """Two ranks, each filtering its row stripe on the GPU (cuda:rank mod
    #devices), stitched on rank 0 == the whole-image reference result."""
    img = np.random.default_rng(6).integers(0, 65536, (203, 171, 3)).astype(np.uint16)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_worker, args=(r, 2, port, img, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert np.array_equal(out, _oracle_fn(img, FilterParams(shape=ShapeSpec("circle", 7))))
