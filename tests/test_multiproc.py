"""World-size-2 (gloo, CPU) coverage of the multi-GPU evidence-batch path
(DESIGN.md §6): contiguous case shards regenerated per rank from
the shared seed, and the single posterior all-gather.  The per-case device step
is stood in for by the oracle here (no GPU on the CI host)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1202_3777_b200 import synth
from paper_1202_3777_b200.batch import gather_posteriors, shard_bounds


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _posteriors(tree, tables, cases):
    from oracle import jtref

    template = jtref.from_potentials(tree, tables)
    return np.stack([jtref.case_posteriors(template, ev, range(len(tree.cards))) for ev in cases])


def _rank_main(rank, world, port, n_cases, out_dir):
    import sys

    sys.path.insert(0, os.path.abspath(os.path.join(os.path.dirname(__file__), "..")))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    tree, tables = synth.make_config("c1")
    lo, hi = shard_bounds(n_cases, world, rank)
    cases = synth.evidence_cases(tree, hi - lo, seed=1234, first=lo)  # only this rank's evidence
    local = torch.from_numpy(_posteriors(tree, tables, cases))
    full = gather_posteriors(local, n_cases)
    if rank == 0:
        np.save(os.path.join(out_dir, "gathered.npy"), full.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("n_cases", [7, 8])
def test_two_rank_shard_and_gather(tmp_path, n_cases):
    port = _free_port()
    mp.spawn(_rank_main, args=(2, port, n_cases, str(tmp_path)), nprocs=2, join=True)
    got = np.load(tmp_path / "gathered.npy")
    tree, tables = synth.make_config("c1")
    want = _posteriors(tree, tables, synth.evidence_cases(tree, n_cases, seed=1234))
    assert got.shape == want.shape
    assert np.array_equal(got, want)  # same computation, same order: bit-identical


@pytest.mark.parametrize("n,world", [(8192, 8), (8191, 8), (5, 4), (3, 2), (0, 2)])
def test_shards_partition_cases(n, world):
    bounds = [shard_bounds(n, world, r) for r in range(world)]
    assert bounds[0][0] == 0 and bounds[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(bounds, bounds[1:]))
    assert max(h - l for l, h in bounds) - min(h - l for l, h in bounds) <= 1
