#!/usr/bin/env python
"""Benchmark of the hot path of arXiv 1808.02950 on B200 (driver contract).

Workload (BASELINE.json config 4, the configuration the metric "8x8 blocks/s
(fwd+retain+inv), achieved HBM GB/s vs B200 peak, 1/2/4/8 GPU" is quoted on): ONE stack of 512
synthetic 3840x2160 8-bit YUV 4:2:0 frames (AR(1) rho = 0.95 luma, rho = 0.9 chroma at half
resolution), sharded by frame over the GPUs (strong scaling; `--scaling weak` gives every GPU
its own 512 frames), forward approximate DCT with the paper's T1 and S, zonal retention r = 10,
inverse, per-frame per-plane SSE and PSNR.  One step = the whole stack (99,532,800 blocks)
through the fused C-ABI call for each plane of each rank's shard + the NCCL all-reduce of the
fp64 [512 x 6] SSE/PSNR table (overlapped with the next step's kernels).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--scaling weak]
    python bench.py --config C5 [--c5-log2 20,22,...,30]      secondary configurations

Prints one JSON line (rank 0).  Inputs (6.37 GB per 512 frames; 0.8 GB per GPU at 8 GPUs) are
larger than the 126 MB L2, so no flush is needed between steps.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "8x8 blocks/s (fwd+retain+inv)"
UNIT = "blocks/s"
R = 10
FRAMES = 512
H, W = 2160, 3840
BLOCKS_PER_FRAME = (H // 8) * (W // 8) + 2 * (H // 16) * (W // 16)  # 194,400
WORKLOAD = ("C4: 512 frames 3840x2160 YUV 4:2:0 u8 (AR(1) rho=0.95 luma / 0.9 chroma), T1 (P:L1116-1130) "
            "with S, fwd -> zig-zag retain r=10 -> inverse -> per-frame per-plane SSE/PSNR")


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """Samples SM clock and throttle reasons with NVML while the timed region runs."""

    REASONS = {
        "gpu_idle": 0x1, "applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
        "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
        "hw_power_brake_slowdown": 0x80, "display_clock_setting": 0x100,
    }

    def __init__(self, index: int, period: float = 0.01):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self.period = period
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM))
                bits = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for name, b in self.REASONS.items():
                    if bits & b and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self._nv:
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        return {"sm_mhz": statistics.median(self.samples) if self.samples else None,
                "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": len(self.samples)}


def make_frames(lo: int, hi: int, device, seed: int = 4):
    """Frames [lo, hi) of the 512-frame C4 stack (synth batches are aligned to global frame
    indices, so a rank's shard equals the same frames of the whole stack)."""
    y, u, v = synth.yuv420_stack(FRAMES, H, W, seed=seed, device=device, batch=8, lo=lo, hi=hi)
    # the two chroma stacks back to back in one allocation: approx_dct8x8_fused_sse_planes then runs
    # U and V as one launch over both image ranges (same geometry)
    uv = torch.empty((2,) + tuple(u.shape), dtype=u.dtype, device=u.device)
    uv[0].copy_(u)
    uv[1].copy_(v)
    del u, v
    return y, uv[0], uv[1]


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_oracle_sample(planes_cpu, budget_s: float = 10.0):
    """The oracle as it stands on a bounded sample of the same workload: whole frames (Y, U, V)
    taken in order from the first frames of the stack (cycling) for ~budget_s of CPU work, once
    on 1 thread and once on every host thread (SURVEY §8(d) oracle timing)."""
    import oracle
    from oracle import matrices as OM

    n_avail = int(planes_cpu[0].shape[0])

    def rate(threads):
        oracle.set_num_threads(threads)
        t0 = time.perf_counter()
        blocks = frames = 0
        while True:
            f = frames % n_avail
            for p in planes_cpu:
                oracle.codec_sse(p[f:f + 1].numpy(), [R], t=OM.T1)
            blocks += BLOCKS_PER_FRAME
            frames += 1
            if time.perf_counter() - t0 > budget_s:
                break
        return blocks / (time.perf_counter() - t0), frames, blocks

    nproc = os.cpu_count() or 1
    v1, f1, b1 = rate(1)
    vn, fn, bn = rate(nproc)
    return {"value": vn, "unit": UNIT, "cores": nproc, "kind": "oracle", "value_1thread": v1,
            "nproc": nproc, "cpu_model": cpu_model(),
            "sample": f"whole C4 frames (Y+U+V, 194,400 blocks each) cycled from the first {n_avail} frames of the "
                      f"same stack, r={R}, T1, oracle/adct_oracle.c by-definition int64/fp64: {fn} frames on {nproc} "
                      f"OpenMP threads and {f1} on 1 thread, ~{budget_s:.0f} s each"}


def run_reference(args):
    """--impl reference: the CPU oracle (this tier's reference arm) on the host cores."""
    from paper_1808_02950_b200 import parallel

    rank, _, world = parallel.env_rank()
    if rank != 0:
        return 0
    import oracle
    from oracle import matrices as OM

    # bounded per-step sample of the same workload: one frame (Y, U, V) per step
    y, u, v = synth.yuv420_stack(1, H, W, seed=4, device="cpu", batch=1)
    planes = [y.numpy(), u.numpy(), v.numpy()]
    for _ in range(args.warmup):
        for p in planes:
            oracle.codec_sse(p, [R], t=OM.T1)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        for p in planes:
            oracle.codec_sse(p, [R], t=OM.T1)
    dt = time.perf_counter() - t0
    value = BLOCKS_PER_FRAME * args.steps / dt
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3, "higher_is_better": True,
        "scaling": getattr(args, "scaling", "strong"),
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample_per_step": "1 frame (Y+U+V, 194,400 blocks)", "matrix": "T1",
                   "r": R},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
                         "sample": "1 frame of the C4 stack per step (Y+U+V), by-definition C oracle"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def issue_roofline(case, ms, clk, dev):
    """Roofline of an ALU-bound line: warp-instructions per step (ncu smsp__inst_executed.sum,
    profiles/ncu_instructions.json via tools/inst_table.py) / step time against the issue peak
    SMs x 4 SMSPs x 1 warp-instruction/clk at the SM clock sampled during the run."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_instructions.json")) as f:
            inst = json.load(f)[case]["warp_inst_per_step"]
    except (OSError, KeyError, ValueError):
        return {"bound": "alu", "achieved": None, "peak": None, "unit": "warp-inst/s", "frac": None,
                "note": "no instruction count recorded (tools/gpu/ncu_inst.sh)"}
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    peak = sms * 4 * (clk.get("sm_mhz") or 1965) * 1e6
    achieved = inst / (ms * 1e-3)
    return {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "warp-inst/s", "frac": achieved / peak,
            "peak_kind": "issue: SMs x 4 SMSP x 1 warp-inst/clk x sampled SM clock", "traffic": None,
            "warp_inst_per_step": inst, "inst_source": "profiles/ncu_instructions.json (ncu, same command)"}


def _timed(fn, steps, warmup, stream, dev):
    """Mean CUDA-event time (ms) of fn() over `steps` launches after `warmup` (one stream)."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(dev.index or 0) as clk:
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize(dev)
    return e0.elapsed_time(e1) / steps, clk.summary()


def run_config(args):
    """Secondary BASELINE.json configurations (parity-test workloads, reported for evidence; the
    driver's headline line is config 4).  One JSON line per (config, matrix)."""
    import oracle
    from oracle import matrices as OM
    from paper_1808_02950_b200 import adct, catalog, parallel

    rank, local, world = parallel.init()
    if world > 1 and args.config not in ("C3", "C5"):
        raise SystemExit("only --config C3 and C5 shard over GPUs (the other secondary configs are 1-GPU lines)")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    hbm_peak, peak_kind = peaks()
    lines = []

    def emit(cfg, matrix, ms, blocks, bytes_per_block, bound, clk, cpu, extra=None, roofline=None):
        # per-GPU HBM roofline: the GPUs of a sharded line each move blocks / n_gpus
        achieved = blocks * bytes_per_block / (ms * 1e-3) / 1e9 / ((extra or {}).get("n_gpus") or 1)
        line = {"metric": METRIC, "value": blocks / (ms * 1e-3), "unit": UNIT, "n_gpus": 1, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "dtype": "f32",
                "data": "synthetic", "config": {"workload": cfg, "matrix": matrix},
                "roofline": roofline or {"bound": bound, "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                                         "frac": achieved / hbm_peak, "peak_kind": peak_kind,
                                         "bytes_per_block": bytes_per_block},
                "clocks": clk, "cpu_baseline": cpu}
        if extra:
            line.update(extra)
        print(json.dumps(line), flush=True)
        lines.append(line)

    def cpu_rate(fn, blocks):
        t0 = time.perf_counter()
        fn()
        return {"value": blocks / (time.perf_counter() - t0), "unit": UNIT, "cores": oracle.num_threads(),
                "kind": "oracle"}

    if args.config in ("C3", "all"):
        # frames sharded by contiguous range over the ranks; the coefficients stay in each rank's
        # HBM, so there is no collective
        n = 1024
        lo, hi = parallel.shard_range(n, rank, world)
        imgs = synth.ar1_stack(n, 1080, 1920, 0.95, seed=3, device=dev, noise_uniform=4.0, batch=16, lo=lo, hi=hi)
        m = adct.Matrix.from_int(catalog.T1, "T1")
        q = torch.empty((hi - lo, 135, 240, 8, 8), dtype=torch.int16, device=dev)
        parallel.barrier()
        ms, clk = _timed(lambda: adct.approx_dct8x8_fwd_quant(m, imgs, 16, q=q, stream=stream), args.steps,
                         args.warmup, stream, dev)
        ms = parallel.max_over_ranks(ms, dev)
        blocks = n * 135 * 240
        if rank == 0:
            nb, _ = oracle.row_scaling(OM.T1)
            smp = imgs[:2].cpu().numpy()
            cpu = cpu_rate(lambda: oracle.quantize(oracle.forward_int(OM.T1, smp), nb, 16), 2 * 135 * 240)
            cpu["sample"] = "first 2 frames, by-definition forward + exact-integer quantiser"
            emit("C3: 1024 frames 1920x1080 u8 AR(1) rho=0.95 + U(-4,4), forward T1 with S folded into a step-16 "
                 f"quantiser -> int16 block-major, frames sharded over {world} GPU(s)", "T1", ms, blocks, 192, "hbm",
                 clk, cpu, {"n_gpus": world, "scaling": "strong"})
        del imgs, q
    if args.config in ("C5", "all"):
        # BASELINE C5: 2^20 .. 2^30 int16 residual blocks, fused forward + inverse (r = 64) with T1
        # and with the exact DCT through the same path; blocks sharded by contiguous range over the
        # ranks with no collective; 2^30 blocks (137 GB) run IN PLACE (recon is src)
        for lg in [int(v) for v in str(args.c5_log2).split(",")]:
            nblk = 1 << lg
            lo, hi = parallel.shard_range(nblk, rank, world)
            in_place = lg >= 29
            x = synth.laplace_range(lo, hi, seed=5, device=dev)
            rec = x if in_place else torch.empty_like(x)
            steps = max(5, min(args.steps, args.steps * (1 << 26) // nblk))
            for name in ("T1", "DCT"):
                m = adct.Matrix.from_int(catalog.T1, "T1") if name == "T1" else adct.Matrix.from_real(
                    catalog.exact_dct(), "DCT")
                parallel.barrier()
                ms, clk = _timed(lambda: adct.approx_dct8x8_roundtrip(m, x, 64, torch.int16, recon=rec,
                                                                      stream=stream), steps, args.warmup, stream, dev)
                ms = parallel.max_over_ranks(ms, dev)
                # r = 64 round trip is the identity after rounding (bit-exact): in place, x must
                # still equal the generated blocks after every step; checked on sampled batches
                if in_place:
                    smp = sorted({0, (hi - lo) // 2, max(0, hi - lo - 4096)})
                    ok = all(torch.equal(x[a0:a0 + 4096],
                                         synth.laplace_range(lo + a0, min(hi, lo + a0 + 4096), seed=5, device=dev))
                             for a0 in smp)
                else:
                    ok = bool(torch.equal(rec, x))
                if rank != 0:
                    continue
                xs = x[:1 << 14].cpu().numpy()
                if name == "T1":
                    n_, s_ = oracle.row_scaling(OM.T1)
                    g_, _ = oracle.synthesis_matrix(oracle.chat_from_int(OM.T1))
                    fn = lambda: oracle.inverse(g_, oracle.scale(oracle.forward_int(OM.T1, xs), s_))  # noqa: E731
                else:
                    g_, _ = oracle.synthesis_matrix(OM.C)
                    fn = lambda: oracle.inverse(g_, oracle.forward_real(OM.C, xs))  # noqa: E731
                cpu = cpu_rate(fn, 1 << 14)
                cpu["sample"] = "2^14 blocks, by-definition forward + inverse"
                emit(f"C5: 2^{lg} int16 Laplace(10) blocks, fused forward + inverse (r=64) -> int16, "
                     f"{'in place' if in_place else 'out of place'}, blocks sharded over {world} GPU(s)", name, ms,
                     nblk, 256, "hbm", clk, cpu,
                     {"roundtrip_bit_exact": ok, "n_gpus": world, "scaling": "strong", "log2_blocks": lg,
                      "in_place": in_place, "steps": steps})
            del x, rec
            torch.cuda.empty_cache()
    if args.config in ("MERIT", "all"):
        # next row f4: Table 4 figures of merit of the nine matrices over 4096 values of rho in
        # (0, 1) — the Fig. 1 coding-gain curves
        from oracle import merit as OMR
        names = catalog.CONFIG2_ORDER
        mats = [adct.Matrix.from_real(catalog.exact_dct(), "DCT") if nm == "DCT" else
                adct.Matrix.from_int(catalog.INTEGER[nm], nm) for nm in names]
        rho = torch.linspace(0.0005, 0.9995, 4096, dtype=torch.float64, device=dev)
        ms, clk = _timed(lambda: adct.merit_batch(mats, rho, stream=stream), args.steps, args.warmup, stream, dev)
        out = adct.merit_batch(mats, rho).cpu().numpy()
        t1, dct = names.index("T1"), names.index("DCT")
        t0 = time.perf_counter()
        chat = OMR.M.c_hat(np.array(catalog.T1).reshape(8, 8))
        for r in rho.cpu().numpy()[:256]:
            OMR.unified_coding_gain(chat, float(r))
        cdt = (time.perf_counter() - t0) / 256
        line = {"metric": "figure-of-merit evaluations/s (4 measures per (matrix, rho))",
                "value": len(names) * 4096 / (ms * 1e-3), "unit": "(matrix, rho)/s", "n_gpus": 1, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "dtype": "f64",
                "data": "the nine matrices of C2", "config": {"workload": "MERIT (next row f4): Table 4 measures of 9 "
                                                              "matrices x 4096 rho (Fig. 1 curves)"},
                "roofline": dict(issue_roofline("MERIT", ms, clk, dev),
                                 note="fp64 8x8 products per thread; one launch of 9 x 4096 threads: latency sized"),
                "clocks": clk, "fig1_max_cg_gap_T1_minus_DCT_dB": float((out[t1, :, 2] - out[dct, :, 2]).max()),
                "cpu_baseline": {"value": 1.0 / cdt, "unit": "(matrix, rho)/s", "cores": 1, "kind": "oracle",
                                 "sample": "256 rho values, C*_g of T1 only (numpy oracle)"}}
        print(json.dumps(line), flush=True)
    if args.config in ("GREEDY", "all"):
        # next row f3: the greedy angle search of §3 (Fig. 2) — D2 = {0,+-1,+-2}^8 with rows 1, 5
        # fixed over all 720 orders (§4.1), and D1 = {0,+-1}^8 over all 8! = 40320 orders (§3.4)
        import itertools
        from oracle import greedy as OG   # CPU baseline leg only
        cexact = np.array(catalog.exact_dct()).reshape(8, 8)
        for name, ent, fixed, orders in (
                ("D2, rows 1,5 fixed, 720 orders", catalog.P2, catalog.GREEDY_FIXED_ROWS,
                 np.array(list(itertools.permutations([1, 2, 3, 5, 6, 7])), dtype=np.int32)),
                ("D1, all 40320 orders", catalog.P1, None,
                 np.array(list(itertools.permutations(range(8))), dtype=np.int32))):
            wsg = torch.empty(adct.lib.adct_greedy_workspace_bytes(len(ent)), dtype=torch.uint8, device=dev)
            ms, clk = _timed(lambda: adct.greedy_search(cexact, ent, orders, fixed=fixed, device=dev, workspace=wsg,
                                                        stream=stream), args.steps, args.warmup, stream, dev)
            mats, status = adct.greedy_search(cexact, ent, orders, fixed=fixed, device=dev, workspace=wsg)
            st = status.cpu().numpy()
            distinct = len({m.tobytes() for m, s_ in zip(mats.cpu().numpy(), st) if s_ == 0})
            srch = OG.Search(ent)
            t0 = time.perf_counter()
            nsmp = 720 if fixed else 200
            for o in orders[:nsmp]:
                srch.solve(tuple(o), fixed)
            cdt = time.perf_counter() - t0
            cand = len(orders) * (8 - len(fixed or {})) * len(ent) ** 8
            line = {"metric": "greedy search: candidate evaluations/s", "value": cand / (ms * 1e-3),
                    "unit": "candidates/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
                    "higher_is_better": True, "dtype": "f64 score / int8 dp4a orthogonality", "data": "exact DCT C",
                    "config": {"workload": f"GREEDY (next row f3): {name}", "feasible": int((st == 0).sum()),
                               "infeasible": int((st == 1).sum()), "distinct_matrices": distinct},
                    "roofline": dict(issue_roofline("GREEDY D2" if fixed else "GREEDY D1", ms, clk, dev),
                                     note="candidate scan: DP4A orthogonality + fp64 score loads"),
                    "clocks": clk,
                    "cpu_baseline": {"value": nsmp * (8 - len(fixed or {})) * len(ent) ** 8 / cdt,
                                     "unit": "candidates/s", "cores": 1, "kind": "oracle",
                                     "sample": f"{nsmp} orders, numpy oracle (memoised orthogonality masks)"}}
            print(json.dumps(line), flush=True)
    if args.config in ("JAM", "all"):
        # next row f2: 16- and 32-point JAM-scaled T1 (§6.2), fused round trip (r = N^2) of int16
        # Laplace residual blocks (the C5 workload at HEVC block sizes), 2^26 8x8-equivalents
        for n in (16, 32):
            nb = (1 << 26) // ((n // 8) ** 2)
            x = synth.laplace_blocks(nb * (n // 8) ** 2, seed=5, device=dev).reshape(nb, n, n)
            rec = torch.empty_like(x)
            ms, clk = _timed(lambda: adct.approx_dct_jam_roundtrip(n, x, n * n, torch.int16, recon=rec, stream=stream),
                             args.steps, args.warmup, stream, dev)
            ok = bool(torch.equal(rec, x))
            from oracle import jam as OJ
            xs = x[:256].cpu().numpy()
            tt = OJ.T16 if n == 16 else OJ.T32
            cpu = cpu_rate(lambda: OJ.recon_n(tt, xs, n * n), 256)
            cpu["sample"] = f"256 blocks of {n}x{n}, by-definition forward + inverse"
            emit(f"JAM{n} (next row f2): {nb} int16 Laplace(10) {n}x{n} blocks, fused T({n}) forward + inverse "
                 f"(r={n * n}) -> int16; value = {n}x{n} blocks/s", f"T({n})", ms, nb, 4 * n * n, "hbm", clk, cpu,
                 {"roundtrip_bit_exact": ok})
            del x, rec
    if args.config in ("SSIM", "all"):
        # next row f1: forward -> retain r=14 -> inverse -> SSIM with 8x8 windows (reading A18) on
        # 128 luma frames of config 4, in ONE kernel (approx_dct8x8_ssim: no reconstruction in
        # HBM); the two-call pipeline (fp32 reconstruction written and re-read) is timed beside it
        n = 128
        y = synth.ar1_stack(n, 2160, 3840, 0.95, seed=4, device=dev, batch=8)
        m = adct.Matrix.from_int(catalog.T1, "T1")
        rec = torch.empty(y.shape, dtype=torch.float32, device=dev)
        ws = torch.empty(adct.workspace_bytes(adct.geom_of(y), 1), dtype=torch.uint8, device=dev)
        out = torch.empty(n, dtype=torch.float64, device=dev)

        def ssim_pipeline():
            adct.approx_dct8x8_roundtrip(m, y, 14, torch.float32, recon=rec, stream=stream)
            adct.ssim_reduce(y, rec, clip=adct.CLIP, workspace=ws, stream=stream)

        ms_pipe, _ = _timed(ssim_pipeline, args.steps, args.warmup, stream, dev)
        ms, clk = _timed(lambda: adct.approx_dct8x8_ssim(m, y, 14, clip=adct.CLIP, ssim=out, workspace=ws,
                                                         stream=stream), args.steps, args.warmup, stream, dev)
        from oracle import ssim as OS
        smp = y[:1, :256, :256].cpu().numpy()
        cpu = cpu_rate(lambda: OS.ssim(smp, smp), 32 * 32)
        cpu["sample"] = "SSIM of one 256x256 crop (oracle windows)"
        emit(f"SSIM (next row f1): {n} luma frames 3840x2160, T1 round trip r=14 + SSIM 8x8 windows in one kernel "
             "(approx_dct8x8_ssim; bytes/block = 64 u8 in, + the neighbour strips' shared block column)", "T1", ms,
             n * 270 * 480, 64, "hbm", clk, cpu,
             {"pipeline_ms": ms_pipe, "pipeline": "approx_dct8x8_roundtrip (fp32 recon in HBM) + ssim_reduce",
              "roofline": dict(issue_roofline("SSIM", ms, clk, dev),
                               note="fp64 window sums + SSIM formula per window (1.06e9 windows per step)")})
        del y, rec
    if args.config in ("C1", "C2", "all"):
        rs = list(range(1, 65))
        if args.config in ("C1", "all"):
            img = synth.ar1_field(1, 512, 512, 0.95, seed=1).to(dev)
            m = adct.Matrix.from_int(catalog.T1, "T1")
            ws = torch.empty(adct.workspace_bytes(adct.geom_of(img), 64), dtype=torch.uint8, device=dev)
            out = torch.empty((1, 64), dtype=torch.float64, device=dev)
            ms, clk = _timed(lambda: adct.approx_dct8x8_fused_sse(m, img, rs, workspace=ws, sse=out, stream=stream),
                             args.steps, args.warmup, stream, dev)
            cpu = cpu_rate(lambda: oracle.codec_sse(img.cpu().numpy(), rs, t=OM.T1), 4096)
            cpu["sample"] = "the same image, r = 1..64"
            emit("C1: one 512x512 AR(1) image, T1, fwd -> retain r -> inv -> PSNR for every r = 1..64", "T1", ms,
                 4096, 64, "hbm", clk, cpu, extra={"note": "one 512x512 image (256 KB): launch-latency bound, "
                                                          "the HBM fraction is not meaningful"})
        if args.config in ("C2", "all"):
            rho, std = synth.config2_params(45, 2)
            imgs = synth.ar1_stack(45, 512, 512, rho, std=std, seed=2, device=dev, batch=15)
            ws = torch.empty(adct.workspace_bytes(adct.geom_of(imgs), 64), dtype=torch.uint8, device=dev)
            out = torch.empty((45, 64), dtype=torch.float64, device=dev)
            mats = [adct.Matrix.from_real(catalog.exact_dct(), "DCT") if nm == "DCT" else
                    adct.Matrix.from_int(catalog.INTEGER[nm], nm) for nm in catalog.CONFIG2_ORDER]

            def all9():
                for mm in mats:
                    adct.approx_dct8x8_fused_sse(mm, imgs, rs, workspace=ws, sse=out, stream=stream)

            ms, clk = _timed(all9, args.steps, args.warmup, stream, dev)
            smp = imgs[:1].cpu().numpy()
            cpu = cpu_rate(lambda: oracle.codec_sse(smp, rs, t=OM.T1), 4096)
            cpu["sample"] = "image 0, T1, r = 1..64"
            emit("C2: 45 AR(1) 512x512 images, r = 1..64 curves for the 9 matrices (T1, C, T2, LO, SDCT, RDCT, "
                 "BAS-2008b, T4, T6) through the same kernel; value counts block x matrix", "all 9", ms,
                 45 * 4096 * 9, 64, "alu", clk, cpu, roofline=issue_roofline("C2", ms, clk, dev))
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="own", choices=["own", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--shard-of", default=None,
                    help="q/W: run only rank q of W's share of the C4 stack on this one GPU (a scaling probe; "
                         "value then counts the whole stack's blocks and is NOT a bench line)")
    ap.add_argument("--planes", action="store_true",
                    help="one approx_dct8x8_fused_sse_planes call per step (Y+U+V); the roofline event then "
                         "brackets the three planes")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong (default, BASELINE C4): one 512-frame stack sharded over the GPUs; "
                         "weak: 512 frames per GPU")
    ap.add_argument("--config", default=None, choices=["C1", "C2", "C3", "C5", "SSIM", "JAM", "GREEDY", "MERIT", "all"],
                    help="secondary BASELINE.json configuration instead of the config-4 headline")
    ap.add_argument("--c5-log2", default="20,22,24,26,28,30",
                    help="comma-separated log2 block counts of the C5 sweep (>= 29 runs in place)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.warmup < 3:
        args.warmup = 3
    if args.config:
        return run_config(args)

    from paper_1808_02950_b200 import adct, catalog, parallel

    rank, local, world = parallel.init()
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    side = torch.cuda.Stream(dev)  # the error-table all-reduce overlaps the next step's kernels
    m = adct.Matrix.from_int(catalog.T1, "T1")
    if args.shard_of:
        # scaling probe on ONE GPU (not a bench line): this process does exactly rank q of W's
        # share of the 512-frame stack, e.g. --shard-of 0/8 = the 64 frames of one rank at 8 GPUs
        q, wq = (int(v) for v in args.shard_of.split("/"))
        n_total = FRAMES
        lo, hi = parallel.shard_range(FRAMES, q, wq)
        planes = make_frames(lo, hi, dev)
    elif args.scaling == "strong":
        # BASELINE C4: ONE 512-frame stack sharded over the ranks, [floor(qN/W), floor((q+1)N/W))
        n_total = FRAMES
        lo, hi = parallel.shard_range(FRAMES, rank, world)
        planes = make_frames(lo, hi, dev)
    else:
        # weak scaling (--scaling weak): every rank owns its own 512-frame stack
        n_total = world * FRAMES
        lo, hi = rank * FRAMES, (rank + 1) * FRAMES
        planes = make_frames(0, FRAMES, dev, seed=4 + 1000 * rank)
    n_local = hi - lo
    torch.cuda.synchronize(dev)
    geoms = [adct.geom_of(p) for p in planes]
    ws = torch.empty(max(adct.planes_workspace_bytes(geoms if args.planes else geoms[1:]),
                         max(adct.workspace_bytes(g, 1) for g in geoms)), dtype=torch.uint8, device=dev)
    # the global per-frame table (fp64, columns SSE Y/U/V, PSNR Y/U/V): the kernels write this
    # rank's rows directly; each step's buffer is all-reduced on the side stream while the next
    # step runs (every entry has exactly one non-zero contributor: bit-identical to one GPU)
    etab = parallel.ErrorTable(n_total, 6, lo, hi, device=dev, buffers=2)

    # per-step events around the dominant kernel, on the launching stream: the luma launch (or with
    # --planes the approx_dct8x8_fused_sse_planes call of the three planes)
    ev_luma = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(args.steps)]
    ev_step = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]  # step boundaries
    outs = [([etab.out(i, b) for i in range(3)], [etab.out(3 + i, b) for i in range(3)]) for b in range(2)]

    def step(k, timed=False):
        buf = k % 2
        etab.before_write(buf)
        if timed:
            ev_luma[k][0].record(stream)
        if (not args.planes):
            # luma (the events' kernel), then both chroma planes in one planes call: U and V lie back
            # to back (make_frames), so the library runs them as one launch
            adct.approx_dct8x8_fused_sse(m, planes[0], [R], workspace=ws, sse=outs[buf][0][0], psnr=outs[buf][1][0],
                                         stream=stream)
            if timed:
                ev_luma[k][1].record(stream)
            adct.approx_dct8x8_fused_sse_planes(m, planes[1:], R, sse=outs[buf][0][1:], psnr=outs[buf][1][1:],
                                                workspace=ws, stream=stream)
        else:
            adct.approx_dct8x8_fused_sse_planes(m, planes, R, sse=outs[buf][0], psnr=outs[buf][1], workspace=ws,
                                                stream=stream)
            if timed:
                ev_luma[k][1].record(stream)
        etab.combine(buf, stream=side)
        return buf

    for k in range(args.warmup):
        last = step(k)
    etab.wait(last)
    torch.cuda.synchronize(dev)
    parallel.barrier()
    torch.cuda.synchronize(dev)
    launches0 = adct.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    profile_range = os.environ.get("ADCT_PROFILE_RANGE") == "1"  # ncu --profile-from-start off
    with ClockSampler(local) as clk:
        if profile_range:
            torch.cuda.profiler.start()
        e0.record(stream)
        ev_step[0].record(stream)
        for k in range(args.steps):
            last = step(k, timed=True)
            ev_step[k + 1].record(stream)
        etab.wait(last)  # the last step's all-reduce is inside the timed region
        e1.record(stream)
        torch.cuda.synchronize(dev)
        if profile_range:
            torch.cuda.profiler.stop()
    launches = adct.launch_count() - launches0
    parallel.barrier()
    total_ms = e0.elapsed_time(e1)
    ms_step = parallel.max_over_ranks(total_ms / args.steps, dev)
    per_step = sorted(ev_step[k].elapsed_time(ev_step[k + 1]) for k in range(args.steps))
    ms_best, ms_median = per_step[0], statistics.median(per_step)
    blocks_total = n_total * BLOCKS_PER_FRAME
    value = blocks_total / (ms_step * 1e-3)
    table = etab.table_of(last)

    # dominant kernel: this rank's luma launch (fused_u8_tc_kernel + its finalize;
    # n_local x 32,400 blocks x 64 algorithmic bytes) -- with --planes the Y+U+V call
    # (n_local x 194,400 blocks) -- averaged over the timed steps
    luma_ms = statistics.mean(a.elapsed_time(b) for a, b in ev_luma)
    luma_blocks = n_local * ((H // 8) * (W // 8) if (not args.planes) else BLOCKS_PER_FRAME)
    luma_bytes = luma_blocks * 64
    hbm_peak, peak_kind = peaks()
    achieved = luma_bytes / (luma_ms * 1e-3) / 1e9
    traffic, ipb = None, None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            nt = json.load(f)["simt" if os.environ.get("ADCT_HOT") == "simt" else "tc"]
            traffic, ipb = nt.get("bytes_per_launch"), nt.get("instructions_per_block")
            if traffic is not None:  # recorded per 512-frame launch of what the kernel covers
                traffic = traffic * n_local / FRAMES if nt.get("covers", "luma") == ("luma" if (not args.planes)
                                                                                    else "yuv") else None
    except Exception:
        pass

    # per-plane PSNR of the first frame of the stack, from the library (finalize kernel, fp64);
    # and, outside the timed region, the same frame under the clip policy of SPEC S:L604 ([0, 255]
    # before the error, reading A6): both metrics are reported
    row0 = table[0].cpu()
    clip0 = {}
    if rank == 0:
        for name, p in zip("YUV", planes):
            _, pc = adct.approx_dct8x8_fused_sse(m, p[:1], [R], clip=adct.CLIP, return_psnr=True)
            clip0[name] = float(pc[0, 0])

    # the same step under the SPEC's metric policy (ADCT_CLIP: reconstruction clipped to [0, 255]
    # before the error, S:L604 / reading A6), after the headline's timed region: the tensor-core
    # kernel's clipped epilogue (tc.cu), Y then U then V; SSE/PSNR into scratch tensors
    clip_line = None
    if not args.planes:
        csse = [torch.empty((p.shape[0], 1), dtype=torch.float64, device=dev) for p in planes]
        cpsnr = [torch.empty((p.shape[0], 1), dtype=torch.float64, device=dev) for p in planes]

        def clip_step():
            for p, a, b in zip(planes, csse, cpsnr):
                adct.approx_dct8x8_fused_sse(m, p, [R], clip=adct.CLIP, workspace=ws, sse=a, psnr=b, stream=stream)

        nclip = max(1, min(args.steps, 50))
        for _ in range(3):
            clip_step()
        torch.cuda.synchronize(dev)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record(stream)
        for _ in range(nclip):
            clip_step()
        c1.record(stream)
        torch.cuda.synchronize(dev)
        clip_ms = parallel.max_over_ranks(c0.elapsed_time(c1) / nclip, dev)
        clip_line = {"policy": "ADCT_CLIP: reconstruction clipped to [0, 255] before the error (SPEC S:L604, "
                               "reading A6), no all-reduce", "steps": nclip, "ms_per_step": clip_ms,
                     "value": blocks_total / (clip_ms * 1e-3), "unit": "blocks/s",
                     "frac_of_hbm": n_local * BLOCKS_PER_FRAME * 64 / (clip_ms * 1e-3) / 1e9 / hbm_peak}

    # end-to-end through the host-buffer C-ABI call (pinned host frames, H2D + D2H inside)
    e2e = None
    if not args.no_e2e:
        host = [p.cpu().pin_memory() for p in planes]
        chunk = 16
        hws = torch.empty(max(adct.host_workspace_bytes(adct.geom_of(h), 1, chunk) for h in host),
                          dtype=torch.uint8, device=dev)
        out = [torch.empty((n_local, 1), dtype=torch.float64).pin_memory() for _ in range(3)]
        pout = [torch.empty((n_local, 1), dtype=torch.float64).pin_memory() for _ in range(3)]

        def e2e_step():
            for i, h in enumerate(host):
                adct.approx_dct8x8_fused_sse_host(m, h, [R], hws, chunk, sse_host=out[i], psnr_host=pout[i],
                                                  stream=stream)

        e2e_step()  # warm-up
        parallel.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            e2e_step()
        dt = parallel.max_over_ranks((time.perf_counter() - t0) / args.e2e_steps, dev)
        for i in range(3):
            assert torch.equal(out[i][:, 0], table[lo:hi, i].cpu()) and torch.equal(pout[i][:, 0],
                                                                                    table[lo:hi, 3 + i].cpu())
        e2e = {"value": blocks_total / dt, "unit": UNIT,
               "h2d_bytes_per_step": int(sum(h.numel() for h in host)),
               "d2h_bytes_per_step": int(6 * n_local * 8), "ms_per_step": dt * 1e3,
               "path": "approx_dct8x8_fused_sse_host (pinned host frames, 2-stream H2D/compute overlap; "
                       "SSE + PSNR tables back to the host)"}
        del host

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_oracle_sample([p[:16].cpu() for p in planes])

    if rank == 0:
        sms = torch.cuda.get_device_properties(dev).multi_processor_count
        clk_mhz = clk.summary()["sm_mhz"] or 1965
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "frames_total": n_total, "frames_per_gpu": n_local,
                       "blocks_per_step": blocks_total, "matrix": "T1", "r": R,
                       "parallelism": f"dp{world} ({'one 512-frame stack' if args.scaling == 'strong' else '512 frames per GPU'}"
                                      f" sharded by frame, fp64 SSE/PSNR table all-reduce overlapped)",
                       "l2": "inputs 6.37 GB per 512 frames > 126 MB L2, no flush"},
            "ms_per_step_best": ms_best, "ms_per_step_median": ms_median,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                         "frac": achieved / hbm_peak, "traffic": traffic, "peak_kind": peak_kind,
                         "frac_vs_8TBs_nominal": achieved / 8000.0,
                         "kernel": ("fused_u8_wtile_kernel<T1Mat,10> (SIMT)" if os.environ.get("ADCT_HOT") == "simt"
                                    else "fused_u8_tc_kernel<T1Mat,10> (tcgen05 kind::i8)") +
                                   (f" + finalize_kernel (luma plane, {luma_blocks:,} blocks x 64 B)" if (not args.planes)
                                    else f" x 3 planes + finalizes (Y+U+V call, {luma_blocks:,} blocks x 64 B)"),
                         "kernel_ms": luma_ms},
            # the whole step (Y + U + V + finalizes + the table combine), rank 0's share
            "roofline_step": {"bound": "hbm", "achieved": n_local * BLOCKS_PER_FRAME * 64 / (ms_step * 1e-3) / 1e9,
                              "peak": hbm_peak, "unit": "GB/s",
                              "frac": n_local * BLOCKS_PER_FRAME * 64 / (ms_step * 1e-3) / 1e9 / hbm_peak},
            "clocks": clk.summary(),
            # issue view of the hot kernel: one warp-instruction per clock per
            # SMSP; roof = SMs x 4 x clock x 32 lanes / (thread-instructions per block, ncu)
            "issue_roofline": None if not ipb else {
                "instructions_per_block": ipb,
                "roof_blocks_per_s": sms * 4 * clk_mhz * 1e6 * 32 / ipb,
                "achieved_blocks_per_s": luma_blocks / (luma_ms * 1e-3),
                "frac": luma_blocks / (luma_ms * 1e-3) / (sms * 4 * clk_mhz * 1e6 * 32 / ipb)},
            "gpu_launches": launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "sse_frame0": {"Y": float(row0[0]), "U": float(row0[1]), "V": float(row0[2])},
            "psnr_frame0_dB": {"Y": float(row0[3]), "U": float(row0[4]), "V": float(row0[5])},
            "psnr_frame0_clipped_dB": clip0,
            "clip_policy": clip_line,
        }
        print(json.dumps(line), flush=True)
    if parallel.env_rank()[2] > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
