#!/usr/bin/env python
"""Benchmark of the hot path: compressed H-matrix-vector product on the B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 4] [--scheme afl]

Workload (BASELINE.json metric "compressed H-matvec GB/s (compressed bytes)"):
config 4 (default) -- Matern nu=1.5, l=0.1 on n=524288 seeded uniform points in
the unit cube, leaf 64, eta 2, SVD truncation 1e-6, AFL-APLR lowrank + AFL
dense leaves (13.9 GB compressed): the largest BASELINE configuration that fits
one B200 and BASELINE's 1/2/4/8-GPU scaling workload, so the N = 1 line and the
scaling runs measure the same matrix.  --config 3 (Laplace sphere n=131072,
1.1 GB) is the single-GPU roofline workload of round 1.  A step is one FP64
product y = A x over the whole matrix (repeated products with fixed x).
Compressed streams are far larger than L2, so no L2 flush is needed between
products.  Bytes per product follow SURVEY 8(d): sum(ceil(N w / 8) + 20) over
codec buffers + 8 k per APLR leaf + 8 n (x) + 8 n (y).

N > 1 (torchrun): block-row partition through the library's partitioned
handle (hcmx_gpu_hmat_create_partitioned), x replicated, the y slices
exchanged by NCCL in-place broadcasts inside the library after every product
(strong scaling: the matrix is fixed).
--impl reference: the reference codec (oracle/_ref, /root/reference
codec.cpp) + the restated matvec glue on all host cores, rank 0 only, on a
bounded row sample (config 4: the first quarter of the rows).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region"""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index, self.proc, self.lines = index, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "20"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(1)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0])); mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def partition_rows(flat, world):
    """the one block-row partitioner (distributed.partition_rows -> the C++
    partitioner behind hcmx_gpu_partition_rows)"""
    from paper_2308_10960_b200.distributed import partition_rows as pr
    return pr(flat, world)


WORKLOADS = {
    "1": ("synthetic (seeded Fibonacci sphere, Laplace kernel, BASELINE config 1)",
          "config1: Laplace sphere n={n}, leaf 64, eta 2, SVD 1e-6, {S}-APLR + {S} dense, y=Ax"),
    "3": ("synthetic (seeded Fibonacci sphere, Laplace kernel, BASELINE config 3)",
          "config3: Laplace sphere n={n}, leaf 64, eta 2, SVD 1e-8, {S}-APLR + {S} dense, y=Ax"),
    "4": ("synthetic (seeded uniform unit cube, Matern nu=1.5 l=0.1, BASELINE config 4)",
          "config4: Matern cube n={n}, leaf 64, eta 2, SVD 1e-6, {S}-APLR + {S} dense, y=Ax"),
}


def workload_strings(cfg, n, scheme):
    data, wl = WORKLOADS[str(cfg)]
    return data, wl.format(n=n, S=scheme.upper())


def step_bytes(flat, row_range=None):
    """SURVEY 8(d) algorithmic bytes of one product (beta = 0)"""
    a, b = row_range or (0, flat.n_rows)
    sel = (flat.row0 >= a) & (flat.row1 <= b)  # the leaves restrict() keeps
    tot = 0
    for l in np.nonzero(sel)[0]:
        b0 = int(flat.buf0[l])
        if flat.kind[l] == 0:
            tot += int(flat.plen[b0]) + 20
        else:
            k = int(flat.rank[l])
            tot += int((flat.plen[b0: b0 + 2 * k] + 20).sum()) + 8 * k
    return tot + 8 * flat.n_cols + 8 * (b - a)


def kernel_bytes(flat, row_range=None):
    """algorithmic bytes per launch of phase A (X streams, sigma, x) and phase B
    (dense + W streams, y) of the handle holding rows `row_range` (every leaf
    overlapping it: phase A whole, phase B the overlapping rows' share)"""
    ra, rb = row_range or (0, flat.n_rows)
    a = bb = 0.0
    for l in range(flat.nleaves):
        r0, r1 = int(flat.row0[l]), int(flat.row1[l])
        ov = min(r1, rb) - max(r0, ra)
        if ov <= 0:
            continue
        frac = ov / (r1 - r0)
        b0 = int(flat.buf0[l])
        if flat.kind[l] == 0:
            bb += (int(flat.plen[b0]) + 20) * frac
        else:
            k = int(flat.rank[l])
            a += int((flat.plen[b0 + k: b0 + 2 * k] + 20).sum()) + 8 * k
            bb += int((flat.plen[b0: b0 + k] + 20).sum()) * frac
    return int(a) + 8 * flat.n_cols, int(bb) + 8 * (rb - ra)


def build_flat(cfg, scheme):
    from paper_2308_10960_b200.hmatrix import build_config
    t0 = time.time()
    flat, info = build_config(cfg, scheme=scheme)
    info["setup_s"] = round(time.time() - t0, 2)
    return flat, info


def cpu_reference_value(flat, threads, budget_s=15.0, max_reps=3):
    """the reference codec (oracle/_ref) + restated matvec glue, timed on host
    cores over a bounded sample (whole matrix, or a row slice if one product
    would exceed the budget)"""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle, RefOracle
    if RefOracle.available():
        impl, kind = RefOracle(), "reference"
    else:
        subprocess.run(["make", "-C", os.path.join(ROOT, "oracle"), os.path.join(ROOT, "oracle", "liboracle.so")],
                       capture_output=True)
        impl, kind = Oracle(), "port"
    fh = flat.host()
    x = np.random.default_rng(0).uniform(-1, 1, fh.n_cols)
    # calibrate on a 1/16 row slice, then pick a sample that fits the budget
    sub = restrict(fh, (0, max(64, fh.n_rows // 16 // 64 * 64)))
    t = time.perf_counter()
    impl.hmat_matvec(sub, 1.0, x, 0.0, np.zeros(fh.n_rows), threads=threads)
    dt = time.perf_counter() - t
    frac = min(1.0, (budget_s / max_reps) / max(dt * 16, 1e-9))
    rows = max(64, int(fh.n_rows * frac) // 64 * 64)
    sample = restrict(fh, (0, rows))
    sb = step_bytes(fh, (0, rows))
    times = []
    for _ in range(max_reps):
        t = time.perf_counter()
        impl.hmat_matvec(sample, 1.0, x, 0.0, np.zeros(fh.n_rows), threads=threads)
        times.append(time.perf_counter() - t)
    best = min(times)
    # one thread on a 1/threads slice of the same sample (T = 1 and T = all)
    rows1 = max(64, rows // max(1, threads) // 64 * 64)
    s1 = restrict(fh, (0, rows1))
    sb1 = step_bytes(fh, (0, rows1))
    t = time.perf_counter()
    impl.hmat_matvec(s1, 1.0, x, 0.0, np.zeros(fh.n_rows), threads=1)
    t1 = time.perf_counter() - t
    # parity of the benched product: the same CPU path over the whole matrix (untimed)
    y_ref = impl.hmat_matvec(fh, 1.0, x, 0.0, np.zeros(fh.n_rows), threads=threads)
    return {"value": sb / best / 1e9, "unit": "GB/s", "cores": threads, "kind": kind,
            "sample": f"rows [0,{rows}) of {fh.n_rows} ({sb / 1e6:.1f} MB compressed), best of {max_reps}, "
                      f"{threads} threads",
            "one_thread": {"value": round(sb1 / t1 / 1e9, 3), "sample": f"rows [0,{rows1}), 1 thread"}}, sb, best, y_ref


def cpu_codec_baseline(threads, nblocks=1024):
    """the reference codec (oracle/_ref, codec.cpp:142-171) on config-2 blocks on the
    host: compress and decompress GB/s (same algorithmic bytes as the GPU codec
    numbers) at 1 thread and at all threads, on a bounded sample of the 4096 blocks"""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle, RefOracle
    impl, kind = (RefOracle(), "reference") if RefOracle.available() else (Oracle(), "port")
    rng = np.random.default_rng(2)
    bs = 4096
    vals = np.sign(rng.standard_normal(nblocks * bs)) * 10 ** rng.uniform(-6, 0, nblocks * bs)
    counts = np.full(nblocks, bs, np.int64)
    res = {"kind": kind, "sample": f"{nblocks} of the 4096 config-2 blocks, eps 1e-6, AFL"}
    for t in sorted({1, threads}):
        n = nblocks if t > 1 else max(64, nblocks // 8)
        v, c = vals[: n * bs], counts[:n]
        t0 = time.perf_counter()
        if kind == "reference":
            e, m, sc, poff, blob, plen = impl.compress_batch(v, c, 1e-6, 0, threads=t)
        else:
            e, m, sc, poff, blob = impl.compress_batch(v, c, 1e-6, 0, threads=t)
            plen = (c * (1 + e + m) + 7) // 8
        tc = time.perf_counter() - t0
        algo = 8 * int(c.sum()) + int((plen + 20).sum())
        t0 = time.perf_counter()
        if kind == "reference":
            impl.decompress_batch(blob, poff, plen, c, 0, e, m, sc, threads=t)
        else:
            impl.decompress_batch(blob, poff, c, 0, e, m, sc, threads=t)
        td = time.perf_counter() - t0
        res[f"threads_{t}"] = {"compress_gbs": round(algo / tc / 1e9, 3), "decompress_gbs": round(algo / td / 1e9, 3)}
    res["cores"] = threads
    return res


def restrict(flat, rr):
    """leaves of a row range (same buffers/blob; oracle ignores unlisted leaves)"""
    from dataclasses import replace
    a, b = rr
    sel = (flat.row0 >= a) & (flat.row1 <= b)
    return replace(flat, row0=flat.row0[sel], row1=flat.row1[sel], col0=flat.col0[sel],
                   col1=flat.col1[sel], kind=flat.kind[sel], rank=flat.rank[sel],
                   buf0=flat.buf0[sel], sig0=flat.sig0[sel])


def codec_microbench(reps=10):
    """BASELINE config 2: 4096 blocks of 64x64, sign * 10^U[-6,0], AFL at 1e-4/1e-6/1e-8.
    Inputs resident in HBM; L2 flushed before every timed call (a 256 MB write
    outside the events), each call bracketed by CUDA events on the stream.
      compress_gbs: hcmx_gpu_codec_compress_device (descriptors and flags stay on
        the device, no read-back), the batched API;
      compress_host_api_gbs: hcmx_gpu_codec_compress (returns host descriptors:
        includes the read-back and its synchronisation);
      decompress_gbs: hcmx_gpu_codec_unpack.
    Algorithmic bytes per SURVEY 8(d): 8N + ceil(N w / 8) + 20 per buffer."""
    import torch
    from paper_2308_10960_b200 import codec
    nb, bs = 4096, 4096
    rng = np.random.default_rng(2)
    vals = np.sign(rng.standard_normal(nb * bs)) * 10 ** rng.uniform(-6, 0, nb * bs)
    d = torch.as_tensor(vals).cuda()
    counts = np.full(nb, bs, np.uint64)
    d_voff = torch.as_tensor((np.arange(nb, dtype=np.int64) * bs)).cuda()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    out = {}

    def timed(fn):
        ts = []
        for _ in range(reps):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 1e3)
        return float(np.median(ts))

    for eps in (1e-4, 1e-6, 1e-8):
        bb = codec.compress_batch(d, counts, eps, codec.Scheme.afl, d_voff=d_voff)
        dec = codec.decompress_batch(bb)
        db = codec.device_batch(d, counts, eps, codec.Scheme.afl)
        codec.compress_device(d, db)
        _, nfix = codec.compress_device_finish(d, db)   # bit-exact completion (no threshold cases here)
        torch.cuda.synchronize()
        pay = int(((counts * bb.desc["bit_width"].astype(np.uint64) + 7) // 8).sum()) + 20 * nb
        algo = 8 * nb * bs + pay
        tcd = timed(lambda: codec.compress_device(d, db))
        tch = timed(lambda: codec.compress_batch(d, counts, eps, codec.Scheme.afl, payload=bb.payload,
                                                 d_voff=d_voff))
        td = timed(lambda: codec.decompress_batch(bb, out=dec))
        pk = _peaks()[0]
        out[f"afl_{eps:g}"] = {"w_bits": int(bb.desc["bit_width"][0]),
                               "compress_gbs": round(algo / tcd / 1e9, 1),
                               "decompress_fp64_gbs": round(8 * nb * bs / td / 1e9, 1),  # FP64 side
                               "compress_host_api_gbs": round(algo / tch / 1e9, 1),
                               "decompress_gbs": round(algo / td / 1e9, 1),
                               "compress_frac": round(algo / tcd / 1e9 / pk, 3),
                               "decompress_frac": round(algo / td / 1e9 / pk, 3),
                               "fixups": int(nfix)}
    out["note"] = "L2 flushed before every call; median of per-call CUDA-event times"
    return out


def run_ours(args, rank, world, local):
    import torch
    import torch.distributed as dist
    from paper_2308_10960_b200.hmatrix import HMatrix
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    flat, info = build_flat(args.config, args.scheme)
    if world > 1:
        # this rank's rows through the library's partitioned handle; the exchange
        # (NCCL in-place broadcasts of the y slices) runs inside the library
        from paper_2308_10960_b200.distributed import PartitionedHMatrix, nccl_comm
        comm, _, _ = nccl_comm()
        H = PartitionedHMatrix(flat, comm)
    else:
        comm = None
        H = HMatrix(flat)
    rep = H.memory()
    n = flat.n_rows
    x = torch.as_tensor(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        # N > 1: local product + exchange, every rank ends with all of y
        H.matvec_device(1.0, x, 0.0, y)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(args.steps):
        step()
    e1.record(stream)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    # per-phase kernel times (roofline) from a second pass of the same K steps
    # with events around each phase: events between the kernels replace their
    # programmatic dependent launch, so the headline pass above runs without them
    # (the board reaches its power cap after ~20 back-to-back config-4 products:
    # a 1 s pause puts this pass in the same power state as the headline pass)
    clk = clocks.stop()
    time.sleep(1.0)
    H.timing(1)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    ms_a, ms_b, calls = H.timing(0)
    launches = H.launches() * args.steps
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    total_bytes = step_bytes(flat)  # whole matrix, once per product
    value = total_bytes * args.steps / (ms / 1e3) / 1e9

    # end to end through the reference-facing call: host x in, host y out
    xh = torch.empty(n, dtype=torch.float64, pin_memory=True)
    xh.copy_(x.cpu())
    yh = torch.zeros(n, dtype=torch.float64, pin_memory=True)
    from paper_2308_10960_b200._lib import check, lib
    e2e_pageable_s = None
    if world == 1:
        for _ in range(args.warmup):
            check(lib().hcmx_gpu_hmat_matvec(H._h, 1.0, xh.data_ptr(), 0.0, yh.data_ptr(), 0))
        # per-call wall times: the host is shared and noisy, so the line
        # reports the median call (the mean is kept beside it)
        per_call = []
        for _ in range(args.steps):
            t = time.perf_counter()
            check(lib().hcmx_gpu_hmat_matvec(H._h, 1.0, xh.data_ptr(), 0.0, yh.data_ptr(), 0))
            per_call.append(time.perf_counter() - t)
        e2e_s = float(np.median(per_call)) * args.steps
        e2e_mean_s = float(np.mean(per_call)) * args.steps
        # the same call from pageable host arrays (an Eigen / numpy caller): the
        # library stages x and y through device buffers itself
        xp, yp = xh.numpy().copy(), np.zeros(n)
        for _ in range(2):
            check(lib().hcmx_gpu_hmat_matvec(H._h, 1.0, xp.ctypes.data, 0.0, yp.ctypes.data, 0))
        per_call = []
        for _ in range(args.steps):
            t = time.perf_counter()
            check(lib().hcmx_gpu_hmat_matvec(H._h, 1.0, xp.ctypes.data, 0.0, yp.ctypes.data, 0))
            per_call.append(time.perf_counter() - t)
        e2e_pageable_s = float(np.median(per_call)) * args.steps
    else:
        # hcmx_gpu_hmat_dist_matvec: host x in, the whole y out on every rank;
        # per-call wall times, max over ranks
        yh_np = np.zeros(n)
        xh_np = xh.numpy()
        for _ in range(args.warmup):
            H.matvec(1.0, xh_np, 0.0, yh_np)
        dist.barrier()
        per_call = []
        for _ in range(args.steps):
            t = time.perf_counter()
            H.matvec(1.0, xh_np, 0.0, yh_np)
            per_call.append(time.perf_counter() - t)
        tt = torch.tensor([float(np.median(per_call)), float(np.mean(per_call))], dtype=torch.float64,
                          device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_s, e2e_mean_s = float(tt[0]) * args.steps, float(tt[1]) * args.steps
    # C5-style multi-RHS products: the 4-right-hand-side arena decodes every
    # field once for 4 columns (same matrix, same bytes; device time per product)
    rhs4 = None
    if world == 1 and not args.no_rhs4:
        H4 = HMatrix(flat, nrhs_block=4)
        X4 = torch.as_tensor(np.random.default_rng(1).uniform(-1, 1, (n, 4))).cuda().contiguous()
        Y4 = torch.zeros(n, 4, dtype=torch.float64, device="cuda")
        for _ in range(args.warmup):
            H4.matmat4_device(1.0, X4, 0.0, Y4)
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            H4.matmat4_device(1.0, X4, 0.0, Y4)
        e1.record(stream)
        torch.cuda.synchronize()
        ms4 = e0.elapsed_time(e1) / args.steps
        flops = 4 * 2.0 * rep.uncompressed_equivalent / 8  # 2 flop per stored FP64 entry and RHS
        fp64_peak = None  # measured DFMA throughput (tools/fp64_peak.cu; MEASURED_PEAKS has no FP64 figure)
        pk = os.path.join(ROOT, "profiles", "r1_fp64_peak.json")
        if os.path.exists(pk):
            fp64_peak = json.load(open(pk)).get("fp64_fma_tflops")
        tf = flops / (ms4 / 1e3) / 1e12
        rhs4 = {"nrhs": 4, "ms_per_product": round(ms4, 4),
                "speedup_vs_4_single": round(4 * (ms / args.steps) / ms4, 3),
                "fp64_tflops": round(tf, 3), "fp64_peak_tflops": fp64_peak,
                "fp64_frac": round(tf / fp64_peak, 3) if fp64_peak else None,
                "note": "matmat4_device: Y = A X for 4 interleaved columns, one decode per field"}
        H4.close()
    cplx = None
    if world == 1 and not args.no_complex:
        cplx = complex_bench(args)
    line = None
    data_s, workload_s = workload_strings(args.config, n, args.scheme)
    if rank == 0:
        peak, peak_src = _peaks()
        ka, kb = kernel_bytes(flat, H.row_range if world > 1 else None)
        per_a = ms_a / max(calls, 1)
        per_b = ms_b / max(calls, 1)
        dom = "phase_b" if per_b >= per_a else "phase_a"
        dom_bytes, dom_ms = (kb, per_b) if dom == "phase_b" else (ka, per_a)
        achieved = dom_bytes / (dom_ms / 1e3) / 1e9 if dom_ms > 0 else 0.0
        traffic = None
        tp = os.path.join(ROOT, "profiles", f"ncu_traffic_c{args.config}.json")
        if os.path.exists(tp):
            traffic = json.load(open(tp)).get(dom)
        cpu, parity = None, None
        if not args.no_cpu_baseline and world == 1:
            cpu, _, _, y_ref = cpu_reference_value(flat, os.cpu_count() or 1)
            # the timed product's y (last step) against the CPU reference path
            y_dev = y.cpu().numpy()
            parity = {"rel_err": float(np.linalg.norm(y_dev - y_ref) / np.linalg.norm(y_ref)),
                      "tol": 1e-12, "vs": f"{cpu['kind']} CPU product over the whole matrix, same x"}
        codec_res = codec_microbench() if (world == 1 and not args.no_codec) else None
        if codec_res is not None and not args.no_cpu_baseline:
            codec_res["cpu_baseline"] = cpu_codec_baseline(os.cpu_count() or 1)
        line = {
            "metric": "compressed H-matvec GB/s (compressed bytes)",
            "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": data_s,
            "config": {"workload": workload_s,
                       "n": n, "leaves": info["leaves"], "dense_leaves": info["dense_leaves"],
                       "lowrank_leaves": info["lowrank_leaves"], "mean_rank": round(info["mean_rank"], 2),
                       "bytes_per_step": total_bytes,
                       "fp64_bytes": int(rep.uncompressed_equivalent),
                       "compression_rate": round(rep.uncompressed_equivalent / max(1, rep.dense_compressed + rep.lowrank_compressed), 3),
                       "l2": "inputs larger than L2 (no flush)", "setup_s": info["setup_s"],
                       "parallelism": f"block-row x{world}" if world > 1 else "single GPU",
                       "matvec_frac_of_peak": round(value / world / peak, 4)},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": peak,
                         "peak_source": peak_src, "unit": "GB/s", "frac": round(achieved / peak, 4),
                         "frac_vs_nominal_8tbs": round(achieved / 8000.0, 4),  # north_star's "~8 TB/s"
                         "traffic": traffic, "algorithmic_bytes_per_launch": dom_bytes,
                         "ms_per_launch": round(dom_ms, 5),
                         "phase_ms": {"phase_a": round(per_a, 5), "phase_b": round(per_b, 5)}},
            "cpu_baseline": cpu,
            "e2e": ({"value": round(total_bytes * args.steps / e2e_s / 1e9, 2), "unit": "GB/s",
                     "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                     "statistic": "median of K per-call wall times",
                     "mean_value": round(total_bytes * args.steps / e2e_mean_s / 1e9, 2),
                     "api": ("hcmx_gpu_hmat_matvec (host pointers, pinned; y crosses PCIe as the kernels write it into mapped host memory)"
                             if world == 1 else
                             "hcmx_gpu_hmat_dist_matvec (host x in, local product + NCCL exchange, whole y out; max over ranks)")}
                    if e2e_s else None),
            "e2e_pageable": ({"value": round(total_bytes * args.steps / e2e_pageable_s / 1e9, 2), "unit": "GB/s",
                              "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                              "statistic": "median of K per-call wall times",
                              "api": "hcmx_gpu_hmat_matvec with pageable host x / y (staged by the library)"}
                             if world == 1 else None),
            "gpu_launches": launches,
            "clocks": clk,
        }
        if parity:
            line["parity"] = parity
        if codec_res:
            line["codec"] = codec_res
        if rhs4:
            line["multi_rhs"] = rhs4
        if cplx:
            line["complex"] = cplx
        print(json.dumps(line), flush=True)
    H.close()
    if world > 1:
        dist.barrier()
        from paper_2308_10960_b200._lib import lib as _lib
        _lib().hcmx_gpu_nccl_comm_destroy(comm)
        dist.destroy_process_group()
    return line


def complex_bench(args, reps=5):
    """BASELINE config 5: Helmholtz exp(i kappa r)/(4 pi r), kappa 16, n = 262144
    sphere points, eps 1e-6, 16 complex right-hand sides U[-1,1] + i U[-1,1],
    through ONE complex arena (ComplexHMatrix: every real / imaginary stream
    decoded once per product of two complex columns, complex combination on the
    device).  FP64-bound: reported as FP64 TFLOP/s executed against
    the measured DFMA peak; parity of one column against the CPU oracle applied
    to the same compressed real / imaginary matrices (checker only, untimed)."""
    import torch
    from paper_2308_10960_b200.hmatrix import ComplexHMatrix, build_config_complex
    t0 = time.time()
    fr, fi, info = build_config_complex("5")
    H = ComplexHMatrix(fr, fi)
    setup = time.time() - t0
    n, r = H.n_rows, 16
    rng = np.random.default_rng(5)
    X = rng.uniform(-1, 1, (n, r)) + 1j * rng.uniform(-1, 1, (n, r))
    Xd = torch.as_tensor(X).cuda()
    Y = torch.empty(n, r, dtype=torch.complex128, device="cuda")
    for _ in range(2):
        H.matmat_device(Xd, Y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        H.matmat_device(Xd, Y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    rep = H.memory()
    # every stored real entry: 2 flops per real right-hand-side slot, 4 slots per
    # product of two complex columns, r / 2 products
    flops = 2.0 * (rep.uncompressed_equivalent / 8) * 4 * (r // 2)
    tf = flops / (ms / 1e3) / 1e12
    pk = os.path.join(ROOT, "profiles", "r1_fp64_peak.json")
    peak = json.load(open(pk)).get("fp64_fma_tflops") if os.path.exists(pk) else None
    out = {"workload": "config5: Helmholtz kappa=16 sphere n=%d, leaf 64, eta 2, eps 1e-6, AFL-APLR, 16 complex RHS" % n,
           "ms_per_16rhs_product": round(ms, 3), "fp64_tflops": round(tf, 3), "fp64_peak_tflops": peak,
           "fp64_frac": round(tf / peak, 3) if peak else None,
           "compressed_bytes": int(rep.algorithmic_bytes), "setup_s": round(setup, 1),
           "note": "one complex arena; per product of two complex columns every stream is decoded once"}
    if not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        from oracle import Oracle
        o, th = Oracle(), os.cpu_count() or 1
        frh, fih = fr.host(), fi.host()
        j = r - 1
        mv = lambda h, v: o.hmat_matvec(h, 1.0, np.ascontiguousarray(v), 0.0, np.zeros(n), threads=th)
        ref = (mv(frh, X[:, j].real) - mv(fih, X[:, j].imag)) + 1j * (mv(frh, X[:, j].imag) + mv(fih, X[:, j].real))
        yj = Y[:, j].cpu().numpy()
        out["parity"] = {"rel_err": float(np.linalg.norm(yj - ref) / np.linalg.norm(ref)), "tol": 1e-12,
                         "vs": "port CPU oracle on the same compressed real / imaginary matrices, column 16"}
    H.close()
    return out


def run_reference(args, rank, world):
    if rank != 0:
        return None
    t0 = time.time()
    # the sample: the whole matrix for configs up to 3, the first quarter of the
    # rows (leaves inside them) for config 4 -- each step stays ~1 s on the host
    row_frac = 0.25 if str(args.config) == "4" else 1.0
    flat, info = build_flat_cpu(args.config, args.scheme, row_frac)
    threads = os.cpu_count() or 1
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from oracle import Oracle, RefOracle
    impl, kind = (RefOracle(), "reference") if RefOracle.available() else (Oracle(), "port")
    n = flat.n_rows
    data_s, workload_s = workload_strings(args.config, n, args.scheme)
    x = np.random.default_rng(0).uniform(-1, 1, n)
    # one step = the product over a row-slice sample sized to ~1 s
    nr = int(n * row_frac) // 64 * 64
    sub = restrict(flat, (0, max(64, nr // 16 // 64 * 64)))
    t = time.perf_counter()
    impl.hmat_matvec(sub, 1.0, x, 0.0, np.zeros(n), threads=threads)
    dt = max(time.perf_counter() - t, 1e-6) * 16
    rows = min(nr, max(64, int(nr * min(1.0, 1.0 / dt)) // 64 * 64))
    sample = restrict(flat, (0, rows))
    sb = step_bytes(flat, (0, rows))
    for _ in range(args.warmup):
        impl.hmat_matvec(sample, 1.0, x, 0.0, np.zeros(n), threads=threads)
    t = time.perf_counter()
    for _ in range(args.steps):
        impl.hmat_matvec(sample, 1.0, x, 0.0, np.zeros(n), threads=threads)
    el = time.perf_counter() - t
    v = sb * args.steps / el / 1e9
    desc = f"rows [0,{rows}) of {n} ({sb / 1e6:.1f} MB compressed) per step, {threads} threads"
    line = {"impl": "reference", "metric": "compressed H-matvec GB/s (compressed bytes)",
            "value": round(v, 3), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(el / args.steps * 1e3, 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": data_s,
            "config": {"workload": workload_s,
                       "n": n, "setup_s": round(time.time() - t0, 1)},
            "cpu_baseline": {"value": round(v, 3), "unit": "GB/s", "cores": threads, "kind": kind,
                             "sample": desc},
            "e2e": {"value": round(v, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return line


def build_flat_cpu(cfg, scheme, row_frac=1.0):
    """reference arm setup: FP64 assembly (torch), then the REFERENCE codec on the
    host (compress for dense leaves, restated APLR glue for lowrank leaves).
    row_frac < 1: only the leaves of rows [0, row_frac n) -- the bounded sample
    the reference arm times -- are assembled and compressed"""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle import Oracle, RefOracle
    from paper_2308_10960_b200 import assemble, problems, tree
    from cpu_hmatrix import Flat
    o = RefOracle() if RefOracle.available() else Oracle()
    s = {"afl": 0, "aflp": 1, "bfl": 2, "dfl": 3}[scheme]
    c = problems.config(cfg)
    pts = problems.make_points(c["geometry"], c["n"], 1)
    ct = tree.build_cluster_tree(pts, c["leaf"])
    lv = tree.build_block_tree(ct, ct, c["eta"])
    if row_frac < 1.0:
        from dataclasses import replace as _rep
        keep = lv.row1 <= int(c["n"] * row_frac) // 64 * 64
        lv = _rep(lv, **{k: getattr(lv, k)[keep] for k in ("row", "col", "admissible", "row0", "row1", "col0", "col1")})
    A = assemble.assemble(pts[ct.i2e], lv, problems.make_kernel(c["kernel"]), c["eps"])
    dense, W, X = A.dense.cpu().numpy(), A.W.cpu().numpy(), A.X.cpu().numpy()
    rows = (lv.row1 - lv.row0).astype(np.int64)
    cols = (lv.col1 - lv.col0).astype(np.int64)
    didx = np.nonzero(A.kind == 0)[0]
    dn = rows[didx] * cols[didx]
    vals = np.concatenate([dense[A.dense_off[l]: A.dense_off[l] + rows[l] * cols[l]] for l in didx])
    if isinstance(o, RefOracle):
        de, dm, dsc, dpo, dblob, dpl = o.compress_batch(vals, dn, c["eps"], s, threads=os.cpu_count())
    else:
        de, dm, dsc, dpo, dblob = o.compress_batch(vals, dn, c["eps"], s, threads=os.cpu_count())
    from oracle import Buf
    bufs, buf0 = [], np.zeros(len(lv), np.int64)
    di = {int(l): i for i, l in enumerate(didx)}
    for l in range(len(lv)):
        buf0[l] = len(bufs)
        if A.kind[l] == 0:
            i = di[l]
            n = (int(dn[i]) * o.bit_width(s, int(de[i]), int(dm[i])) + 7) // 8
            bufs.append(Buf(s, int(de[i]), int(dm[i]), float(dsc[i]), int(dn[i]),
                            dblob[int(dpo[i]): int(dpo[i]) + n].tobytes()))
        else:
            k = int(A.rank[l])
            if k:
                Wl = W[A.w_off[l]: A.w_off[l] + rows[l] * k].reshape(k, rows[l]).T
                Xl = X[A.x_off[l]: A.x_off[l] + cols[l] * k].reshape(k, cols[l]).T
                bufs.extend(o.aplr_compress(Wl, Xl, A.sigma[A.sig_off[l]: A.sig_off[l] + k], c["eps"], s))
    poff = np.zeros(len(bufs), np.int64)
    parts, off = [], 0
    for i, b in enumerate(bufs):
        poff[i] = off
        parts.append(np.frombuffer(b.payload, np.uint8))
        off += len(b.payload)
    sig0 = A.sig_off.copy()
    sig0[sig0 < 0] = 0
    flat = Flat(c["n"], c["n"], lv.row0.astype(np.int64), lv.row1.astype(np.int64),
                lv.col0.astype(np.int64), lv.col1.astype(np.int64), A.kind.astype(np.int64),
                A.rank.astype(np.int64), buf0, sig0, A.sigma, np.array([b.scheme for b in bufs], np.uint8),
                np.array([b.e for b in bufs], np.uint8), np.array([b.m for b in bufs], np.uint8),
                np.array([b.scale for b in bufs]), np.array([b.count for b in bufs], np.int64), poff,
                np.array([len(b.payload) for b in bufs], np.int64), np.concatenate(parts))
    flat.nleaves = len(lv)
    return flat, {}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="4")
    ap.add_argument("--scheme", default="afl", choices=["afl", "aflp", "bfl", "dfl"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-codec", action="store_true")
    ap.add_argument("--no-rhs4", action="store_true")
    ap.add_argument("--no-complex", action="store_true", help="skip the config-5 complex multi-RHS measurement")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)


if __name__ == "__main__":
    main()
