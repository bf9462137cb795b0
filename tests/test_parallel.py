"""Multi-process plumbing of the sharded path on CPU (gloo, world size 2 and 3).

The path shards images over ranks with no data exchange (every 8x8 block, hence every image,
is independent: PAPER.md §6.1); the only collective is the all-reduce of the
per-image error table, in which every entry has exactly one non-zero contributor, so the
combined table must equal the single-process table bit for bit.  The per-image sums here
come from the CPU oracle (the CUDA path is covered by the -m gpu tests); what is tested is
the sharding arithmetic and the collective.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1808_02950_b200 import parallel


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_shard_range_partitions():
    for n in (0, 1, 5, 45, 512, 1000):
        for world in (1, 2, 3, 4, 8):
            spans = [parallel.shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and a <= b
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        parallel.shard_range(4, 2, 2)


def _worker(rank, world, port, tables, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    try:
        r, _, w = parallel.init(backend="gloo")
        assert (r, w) == (rank, world)
        full = torch.from_numpy(tables)
        n = full.shape[0]
        lo, hi = parallel.shard_range(n, rank, world)
        local = torch.zeros_like(full)
        local[lo:hi] = full[lo:hi]                      # this rank filled only its own images
        parallel.combine_error_table(local)
        # the bench's per-step pattern: combined again and again, the table must not drift
        et = parallel.ErrorTable(n, full.shape[1], lo, hi)
        for _ in range(3):
            for c in range(full.shape[1]):
                et.set_local(c, full[lo:hi, c])
            tab = et.combine()
        stable = tab.numpy().tobytes() == full.numpy().tobytes()
        t = parallel.max_over_ranks(float(rank) + 0.5)
        parallel.barrier()
        q.put((rank, local.numpy().tobytes() == full.numpy().tobytes() and stable, t))
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_error_table_allreduce_is_bit_identical(world):
    import oracle
    from oracle import matrices as OM
    import synth

    imgs = synth.ar1_field(5, 32, 48, [0.86, 0.9, 0.95, 0.97, 0.98], seed=11).numpy()
    tables = oracle.codec_sse(imgs, [1, 3, 10, 36, 64], t=OM.T1)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, tables, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _ in res)
    assert all(t == world - 0.5 for _, _, t in res)  # max over ranks


def test_error_table_out_views_are_contiguous_rank_rows():
    """ErrorTable.out(col) is where a kernel writes one column of this rank's rows: contiguous,
    aliasing `local`, and combine() returns the [n_total, cols] table."""
    et = parallel.ErrorTable(10, 3, 4, 7)
    for c in range(3):
        o = et.out(c)
        assert o.is_contiguous() and o.shape == (3,)
        o.copy_(torch.arange(3, dtype=torch.float64) + 10 * c)
    tab = et.combine()
    assert tab.shape == (10, 3)
    assert torch.equal(tab[4:7], et.local[4:7])
    assert torch.equal(tab[4:7, 2], torch.tensor([20.0, 21.0, 22.0], dtype=torch.float64))
    assert float(tab[:4].abs().sum()) == 0.0 and float(tab[7:].abs().sum()) == 0.0
