"""Multi-GPU plumbing: one process per GPU, images (frames) sharded over ranks.

The path partitions naturally: every 8x8 block — hence every image — is processed
independently (§6.1; "no inter-block state"), so ranks never exchange
pixels.  The only collective is the one the north star names: the per-image error table
(fp64 [n_images, n_r]) is combined with an all-reduce(SUM) in which each entry has exactly
one non-zero contributor, so the combined table is bit-identical to a 1-GPU run.
"""
from __future__ import annotations

import os

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous share [lo, hi) of n items for `rank` of `world`: floor(q n / W) boundaries."""
    if world < 1 or not (0 <= rank < world) or n < 0:
        raise ValueError("bad shard arguments")
    return (rank * n) // world, ((rank + 1) * n) // world


def env_rank() -> tuple[int, int, int]:
    """(rank, local_rank, world_size) from the torchrun environment (1 process if unset)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("LOCAL_RANK", "0")),
            int(os.environ.get("WORLD_SIZE", "1")))


def init(backend: str | None = None) -> tuple[int, int, int]:
    """Process group for torchrun ranks (NCCL over NVLink when CUDA is available).

    Test hooks: ADCT_DIST_BACKEND overrides the backend; ADCT_ONE_DEVICE=1 puts every rank on
    cuda:0 (with the gloo backend) so that the multi-rank host logic of bench.py can run on a
    single-GPU box — the ranks' kernels never wait on each other, only host collectives do."""
    rank, local, world = env_rank()
    if os.environ.get("ADCT_ONE_DEVICE") == "1":
        local = 0
    backend = backend or os.environ.get("ADCT_DIST_BACKEND") or None
    if world > 1 and not dist.is_initialized():
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group(backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, local, world


class ErrorTable:
    """The global per-image error table [n_total, cols] (fp64) of a sharded run.

    `local` holds this rank's rows [lo, hi) and zeros elsewhere; `combine()` copies it into the
    output and all-reduces (SUM), so every entry has exactly one non-zero contributor and the
    result is bit-identical to a single-process run however often it is combined.  (All-reducing
    the output in place step after step would add the other ranks' stale copies.)  Storage is
    column-major, so `out(col)` -- this rank's rows of one column -- is contiguous and a kernel
    writes its per-image results there directly; `local` and `table` are [n_total, cols] views.

    With buffers=2 and a side stream, step k writes buffer k % 2 while the previous step's
    buffer is copied and all-reduced on the side stream (`combine(buf, stream=side)`), so the
    collective overlaps the next step's kernels; `before_write(buf)` orders the rewrite of a
    buffer after its last copy and `wait(buf)` orders the current stream after its all-reduce."""

    def __init__(self, n_total: int, cols: int, lo: int, hi: int, device=None, buffers: int = 1):
        self.lo, self.hi = lo, hi
        self._local = torch.zeros((buffers, cols, n_total), dtype=torch.float64, device=device)
        self._table = torch.zeros_like(self._local)
        self._copied = [None] * buffers
        self._done = [None] * buffers
        self.local = self._local[0].t()
        self.table = self._table[0].t()

    def out(self, col: int, buf: int = 0) -> torch.Tensor:
        return self._local[buf, col, self.lo:self.hi]

    def local_of(self, buf: int) -> torch.Tensor:
        return self._local[buf].t()

    def table_of(self, buf: int) -> torch.Tensor:
        return self._table[buf].t()

    def set_local(self, col: int, values: torch.Tensor, buf: int = 0) -> None:
        self.out(col, buf).copy_(values.reshape(self.hi - self.lo))

    def combine(self, buf: int = 0, stream=None) -> torch.Tensor:
        if stream is None:
            self._table[buf].copy_(self._local[buf])
            combine_error_table(self._table[buf])
            return self.table_of(buf)
        cur = torch.cuda.current_stream(self._local.device)
        stream.wait_stream(cur)  # after the kernels that wrote this buffer
        if self._copied[buf] is None:
            self._copied[buf] = torch.cuda.Event()
            self._done[buf] = torch.cuda.Event()
        with torch.cuda.stream(stream):
            self._table[buf].copy_(self._local[buf])
            self._copied[buf].record(stream)
            combine_error_table(self._table[buf])
            self._done[buf].record(stream)
        return self.table_of(buf)

    def before_write(self, buf: int) -> None:
        if self._copied[buf] is not None:
            torch.cuda.current_stream(self._local.device).wait_event(self._copied[buf])

    def wait(self, buf: int) -> None:
        if self._done[buf] is not None:
            torch.cuda.current_stream(self._local.device).wait_event(self._done[buf])


def combine_error_table(local: torch.Tensor) -> torch.Tensor:
    """All-reduce(SUM) of a per-image error table whose rows outside this rank's shard are 0."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(local, op=dist.ReduceOp.SUM)
    return local


def max_over_ranks(value: float, device=None) -> float:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        t = torch.tensor([value], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    return value


def barrier() -> None:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.barrier()
