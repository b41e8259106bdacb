"""CPU, world_size 2 over gloo: the multi-rank estimator path (contiguous
sample shards per rank, per-sample slot buffers, one all-reduce per level,
fixed-order reduction) gives results bitwise identical to one rank
(SPEC.md:313 execution-order independence)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2507_19246_b200.mlmc import FixedSamples, mlmc_estimate
from paper_2507_19246_b200.models import make_hierarchy, toy_family

COUNTS = (37, 11, 5)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out, cap=None):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        fam = toy_family(make_hierarchy([0.1, 0.05, 0.025]), cap=cap)
        res = mlmc_estimate(fam, policy=FixedSamples(COUNTS), seed=11)
        out[rank] = (res.expectation, [(s.sum_y, s.sum_y2, s.n) for s in res.per_level])
    finally:
        dist.destroy_process_group()


def run(world, cap=None):
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, port, out, cap), nprocs=world, join=True)
    return dict(out)


@pytest.mark.timeout(180)
def test_two_ranks_bitwise_equal_one_rank():
    one = run(1)[0]
    two = run(2)
    assert two[0] == two[1]                 # every rank holds the same estimate
    assert two[0] == one                    # and it equals the single-rank result
    fam = toy_family(make_hierarchy([0.1, 0.05, 0.025]))
    local = mlmc_estimate(fam, policy=FixedSamples(COUNTS), seed=11)
    assert local.expectation == one[0]


@pytest.mark.timeout(180)
def test_two_ranks_chunked_path_bitwise_equal_one_rank():
    """The chunked estimator path (_run_chunked: each rank's samples in
    run_levels calls of <= cap samples per level, as full-size streaming
    configs run) under a 2-rank gloo group equals the unchunked 1-rank
    estimate bitwise (parareal.py:185-188 worker-count independence)."""
    one = run(1)[0]
    two = run(2, cap=4)
    assert two[0] == two[1]
    assert two[0] == one
