"""Sharded CUDA path in several processes (row a10 / §8(e)): frames split by contiguous range
over the ranks, each rank runs the fused C-ABI call on its shard and writes SSE and PSNR into
its rows of the global table, and the table is combined with an all-reduce (NCCL when every rank
has its own GPU, else gloo with every rank on cuda:0 -- ADCT_ONE_DEVICE=1; the ranks' kernels
never wait on each other, only the host collective does).  The combined table must equal the
1-process table bit for bit and the oracle on every frame (blocks are
independent and the per-image reduction is order-independent of the sharding).

The double-buffered side-stream combine of bench.py (ErrorTable(buffers=2).combine(buf,
stream=side)) is the path exercised.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from oracle import matrices as M
import synth

pytestmark = pytest.mark.gpu

N_FRAMES = 7
SHAPES = {"Y": (1088, 1920), "U": (544, 960)}  # H, W multiples of 8


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _stack(lo, hi):
    y = synth.ar1_stack(N_FRAMES, *SHAPES["Y"], 0.95, seed=61, batch=2, lo=lo, hi=hi)
    u = synth.ar1_stack(N_FRAMES, *SHAPES["U"], 0.90, seed=62, batch=2, lo=lo, hi=hi)
    return [y, u]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    two_gpus = torch.cuda.device_count() >= world
    if not two_gpus:
        os.environ["ADCT_ONE_DEVICE"] = "1"
    try:
        from paper_1808_02950_b200 import adct, catalog, parallel
        r, local, w = parallel.init(backend="nccl" if two_gpus else "gloo")
        dev = torch.device("cuda", local)
        stream = torch.cuda.current_stream(dev)
        side = torch.cuda.Stream(dev)
        m = adct.Matrix.from_int(catalog.T1, "T1")
        lo, hi = parallel.shard_range(N_FRAMES, r, w)
        planes = [p.to(dev) for p in _stack(lo, hi)]
        et = parallel.ErrorTable(N_FRAMES, 2 * len(planes), lo, hi, device=dev, buffers=2)
        last = 0
        for k in range(4):  # the bench's step pattern: alternate buffers, combine on the side stream
            buf = k % 2
            et.before_write(buf)
            if hi > lo:
                for i, p in enumerate(planes):
                    adct.approx_dct8x8_fused_sse(m, p, [10], sse=et.out(i, buf), psnr=et.out(len(planes) + i, buf),
                                                 stream=stream)
            et.combine(buf, stream=side)
            last = buf
        et.wait(last)
        torch.cuda.synchronize(dev)
        q.put((r, et.table_of(last).cpu().numpy()))
    except Exception as e:  # report instead of hanging the parent
        q.put((rank, repr(e)))
        raise
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()


def _run(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0, res
    return res


@pytest.fixture(scope="module")
def one_rank_table():
    from paper_1808_02950_b200 import adct, catalog
    m = adct.Matrix.from_int(catalog.T1, "T1")
    cols = []
    psnrs = []
    for p in _stack(0, N_FRAMES):
        sse, psnr = adct.approx_dct8x8_fused_sse(m, p.cuda(), [10], return_psnr=True)
        cols.append(sse.cpu().numpy()[:, 0])
        psnrs.append(psnr.cpu().numpy()[:, 0])
    return np.stack(cols + psnrs, axis=1)


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_table_equals_one_rank_and_oracle(world, one_rank_table):
    res = _run(world)
    tabs = list(res.values())
    assert all(isinstance(t, np.ndarray) for t in tabs), res
    for t in tabs:  # every rank holds the same combined table, equal to 1 process bit for bit
        assert t.tobytes() == one_rank_table.tobytes()
    planes = _stack(0, N_FRAMES)
    for i, p in enumerate(planes):
        ref = oracle.codec_sse(p.numpy(), [10], t=M.T1)[:, 0]
        got = one_rank_table[:, i]
        assert np.all(np.abs(got - ref) <= 1e-5 * ref)
        npix = p.shape[1] * p.shape[2]
        for f in range(N_FRAMES):
            assert abs(one_rank_table[f, len(planes) + i] - oracle.psnr(ref[f], npix)) <= 1e-3


@pytest.mark.skipif(not torch.cuda.is_available() or torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_second_device_after_first():
    """Per-device lazy setup (function attributes, the sweep kernel's __constant__ zig-zag table,
    the host pipeline's copy stream): the same calls on cuda:1 after cuda:0 give the same results
    (ADVICE r1)."""
    from paper_1808_02950_b200 import adct, catalog
    m = adct.Matrix.from_int(catalog.T1, "T1")
    img = synth.ar1_field(2, 64, 256, 0.95, seed=8)
    out = []
    for d in (0, 1):
        with torch.cuda.device(d):
            x = img.to(f"cuda:{d}")
            sweep = adct.approx_dct8x8_fused_sse(m, x, [1, 10, 30]).cpu()      # sweep kernel (c_zz)
            hot = adct.approx_dct8x8_fused_sse(m, x, [10]).cpu()               # tensor-core kernel
            rt = adct.approx_dct8x8_roundtrip(m, x[:, :, :64].contiguous(), 10, torch.int16).cpu()
            host = img.pin_memory()
            ws = torch.empty(adct.host_workspace_bytes(adct.geom_of(host), 1, 1), dtype=torch.uint8,
                             device=f"cuda:{d}")
            h = adct.approx_dct8x8_fused_sse_host(m, host, [10], ws, chunk_images=1)
            out.append((sweep, hot, rt, h))
    for a, b in zip(out[0], out[1]):
        assert torch.equal(a, b)
