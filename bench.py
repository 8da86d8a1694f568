#!/usr/bin/env python
"""bench.py -- cuSZ+ compress/decompress throughput on B200 (driver contract).

One STEP = one compress + one decompress of the workload field, device
resident (``compress_device`` -> ``decompress_device``), archives bit-exact
with the CPU reference.  Default workload (BASELINE.json configs[4], the
north-star config; it fits one B200): C5 = 2048^3 float32 synthetic smooth
field (SURVEY 8(d) generator), rel eb 1e-4, auto workflow (-> Huffman).
Inputs (34 GB) are far larger than L2 (126 MB), so no flush is needed.

  value       uncompressed GB/s of the round trip: N*4 / (t_compress + t_decompress)
  compress_gbs / decompress_gbs   the two directions separately (paper style)
  roofline    dominant kernel: algorithmic bytes / CUDA-event time vs the
              measured HBM copy peak (MEASURED_PEAKS.json)
  e2e         same metric through the public API with HOST (pinned) buffers:
              H2D field, compress, D2H archive, H2D archive, decompress, D2H field;
              consecutive steps pipelined over two copy streams (full-duplex PCIe)
  cpu_baseline  the CPU oracle port (oracle/, 1 thread) on a bounded sub-slab

--impl reference: the reference's CPU algorithm (the oracle port; the Python
reference cannot travel to the GPU box) on all host threads, per-step sample
of the same workload; rank 0 only.

Multi-GPU (torchrun, N>1): strong scaling of the same 2048^3 field cut into
N z-slabs of whole chunk layers (paper_2105_12912_b200.distributed): per rank
K1 on its slab, NCCL all-reduce of the 8 KB histogram, identical K2 code book,
all-gather of (bits, outliers) for archive offsets, K3 at the slab's bit
phase.  Time = max over ranks (CUDA events).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "compress/decompress GB/s at 1-8 B200 (% of HBM roofline) + compression ratio"

CONFIGS = {
    "c5": dict(shape=(2048, 2048, 2048), gen="smooth", eb=1e-4,
               workload="C5: 3D float32 2048x2048x2048 synthetic smooth field, rel eb 1e-4"),
    "c5s": dict(shape=(512, 512, 512), gen="smooth", eb=1e-4,
                workload="C5s: 3D float32 512^3 smooth (C5 per-element behaviour, profiling size)"),
    "c5q": dict(shape=(512, 2048, 2048), gen="smooth", eb=1e-4,
                workload="C5q: 3D float32 512x2048x2048 smooth (C5 per-element and decode-layout behaviour, profiling size)"),
    "c1": dict(shape=(100, 500, 500), gen="smooth", eb=1e-4,
               workload="C1: 3D float32 100x500x500 (Hurricane shape) smooth, rel eb 1e-4"),
    "c2": dict(shape=(1800, 3600), gen="smooth", eb=1e-4,
               workload="C2: 2D float32 1800x3600 (CESM shape) smooth, rel eb 1e-4"),
    "c3": dict(shape=(280953867,), gen="smooth1d", eb=1e-4,
               workload="C3: 1D float32 280953867 (HACC shape) smooth, rel eb 1e-4"),
    "c4": dict(shape=(512, 512, 512), gen="sparse", eb=1e-2,
               workload="C4: 3D float32 512^3 (Nyx shape) sparse, rel eb 1e-2 (RLE+VLE)"),
}


# ---------------------------------------------------------------------------
# synthetic fields, generated on the device slab by slab
# ---------------------------------------------------------------------------
def gen_smooth_device(shape, z0, z1, device, ramp=True):
    import torch

    nd = len(shape)
    f64 = torch.float64
    if nd == 1:
        (nx,) = shape
        out = torch.empty(z1 - z0, dtype=torch.float32, device=device)
        step = 1 << 26
        for a in range(z0, z1, step):
            b = min(z1, a + step)
            x = torch.arange(a, b, dtype=f64, device=device)
            d = torch.sin(x / 13.0) * 40.0
            if ramp:
                d = d + 0.03 * x
            out[a - z0: b - z0] = d.to(torch.float32)
        return out
    if nd == 2:
        ny, nx = shape
        y = torch.arange(z0, z1, dtype=f64, device=device)
        x = torch.arange(nx, dtype=f64, device=device)
        d = (torch.sin(y / 13.0)[:, None] + torch.sin(x / 20.0)[None, :]) * 40.0
        if ramp:
            d = d + 0.03 * x[None, :]
        return d.to(torch.float32).reshape(-1)
    nz, ny, nx = shape
    out = torch.empty((z1 - z0, ny, nx), dtype=torch.float32, device=device)
    y = torch.arange(ny, dtype=f64, device=device)
    x = torch.arange(nx, dtype=f64, device=device)
    sy = torch.sin(y / 20.0)
    sx = torch.sin(x / 27.0)
    rx = 0.03 * x
    for za in range(z0, z1, 16):
        zb = min(z1, za + 16)
        z = torch.arange(za, zb, dtype=f64, device=device)
        sz = torch.sin(z / 13.0)
        d = ((sz[:, None, None] + sy[None, :, None]) + sx[None, None, :]) * 40.0
        if ramp:
            d = d + rx[None, None, :]
        out[za - z0: zb - z0] = d.to(torch.float32)
    return out.reshape(-1)


def gen_sparse_device(shape, device, seed=0):
    import numpy as np
    import torch

    rng = np.random.default_rng(seed)
    data = torch.full(shape, 1.0, dtype=torch.float64, device=device)
    nblobs = max(8, int(np.prod(shape) // 2_000_000))
    for _ in range(nblobs):
        c = [rng.uniform(0, s) for s in shape]
        w = rng.uniform(2.0, 6.0)
        amp = float(np.exp(rng.normal(3.0, 1.0)))
        lo = [max(0, int(ci - 4 * w)) for ci in c]
        hi = [min(s, int(ci + 4 * w) + 1) for ci, s in zip(c, shape)]
        axes = [torch.arange(a, b, dtype=torch.float64, device=device) - ci
                for a, b, ci in zip(lo, hi, c)]
        r2 = sum(g.reshape([-1 if k == i else 1 for k in range(len(shape))]) ** 2
                 for i, g in enumerate(axes))
        sl = tuple(slice(a, b) for a, b in zip(lo, hi))
        data[sl] += amp * torch.exp(-r2 / (2 * w * w))
    return data.to(torch.float32).reshape(-1)


def gen_field_device(cfg, device, z0=None, z1=None):
    shape = cfg["shape"]
    if cfg["gen"] == "sparse":
        return gen_sparse_device(shape, device)
    lead = shape[0]
    z0 = 0 if z0 is None else z0
    z1 = lead if z1 is None else z1
    return gen_smooth_device(shape, z0, z1, device, ramp=cfg["gen"] != "smooth1d")


def gen_sample_host(cfg, planes):
    """Host numpy sub-slab of the workload for the CPU legs (same generator)."""
    import numpy as np

    shape = list(cfg["shape"])
    if cfg["gen"] == "sparse":
        return gen_sparse_device(tuple(shape), "cpu").numpy(), tuple(shape)
    shape[0] = min(shape[0], planes)
    axes = [np.arange(n, dtype=np.float64) for n in shape]
    g = np.meshgrid(*axes, indexing="ij", sparse=True)
    data = np.zeros(shape, np.float64)
    for i, a in enumerate(g):
        data = data + np.sin(a / (13.0 + 7 * i))
    data = data * 40.0
    if cfg["gen"] != "smooth1d":
        data = data + 0.03 * g[-1]
    return data.astype(np.float32).reshape(-1), tuple(shape)


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md)
# ---------------------------------------------------------------------------
class ClockSampler:
    Q = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = os.path.join(ROOT, "gpurun_out", f"clocks_rank{gpu_index}.csv")

    def start(self):
        self.t0 = self.t1 = None
        try:
            os.makedirs(os.path.dirname(self.path), exist_ok=True)
            self.fh = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=self.fh, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None
        time.sleep(1.5)  # nvidia-smi start-up; the first samples precede the timed region

    def mark(self, which):
        from datetime import datetime

        setattr(self, which, datetime.now())

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.3)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.fh.close()
        from datetime import datetime

        rows, allrows = [], []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                ts = datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f")
                row = (float(parts[1]), float(parts[2]), parts[5:9])
            except ValueError:
                continue
            allrows.append(row)
            if self.t0 and self.t1 and self.t0 <= ts <= self.t1:
                rows.append(row)
        if not rows:
            rows = allrows[-3:]  # timed region shorter than the sampling period
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for _, _, flags in rows for k, f in enumerate(flags)
                          if f.lower() == "active"})
        loaded = [r[0] for r in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(r[1] for r in rows),
                "reasons": reasons, "samples": len(rows)}


# ---------------------------------------------------------------------------
def measured_peak_hbm():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


def profiled_traffic(kernel: str):
    """dram bytes per launch from the committed ncu --set full capture, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(p) as fh:
            return json.load(fh).get(kernel)
    except (OSError, ValueError):
        return None


# kernels each C-ABI call launches (ours only; memsets/copies excluded), used
# for the gpu_launches claim and cross-checked by the committed ncu launch list
# our kernels per C-ABI call on the C5 path (k_mm_init included)
# kernels per call, as in the ncu launch list of one bench step (profiles/r2g_launches_c5.csv)
LAUNCHES = {"lzb_quantize": 8, "lzb_codebook": 1, "lzb_huff_encode": 4, "lzb_huff_decode": 5,
            "lzb_reconstruct_with_outliers": 7, "lzb_reconstruct_no_outliers": 5,
            "lzb_rle_encode": 6, "lzb_histogram": 1, "lzb_rle_decode": 3,
            "status_and_header_copies": 5}  # k_copy_bytes: 3 status reads + 2 header writes


def launches_per_step(header) -> int:
    from paper_2105_12912_b200 import Workflow

    n = LAUNCHES["lzb_quantize"] + LAUNCHES["lzb_codebook"] + LAUNCHES["status_and_header_copies"]
    if header.workflow is Workflow.HUFFMAN:
        n += LAUNCHES["lzb_huff_encode"] + LAUNCHES["lzb_huff_decode"]
        if header.count <= (1 << 25):  # single-sync compress: + the device archive assembly
            n += 1
    elif header.workflow is Workflow.RLE:
        n += LAUNCHES["lzb_rle_encode"] + LAUNCHES["lzb_rle_decode"]
    else:
        n += (LAUNCHES["lzb_rle_encode"] + LAUNCHES["lzb_histogram"] + LAUNCHES["lzb_codebook"]
              + LAUNCHES["lzb_huff_encode"] + LAUNCHES["lzb_huff_decode"]
              + LAUNCHES["lzb_rle_decode"])
    n += LAUNCHES["lzb_reconstruct_with_outliers" if header.outlier_count
                  else "lzb_reconstruct_no_outliers"]
    return n


def stage_bytes(name, n, s, arc_bits_bytes, n_out):
    """Algorithmic bytes per launch of each stage."""
    return {
        "K1_quantize": n * s + n * 2 + 16 * n_out,
        "K3_huff_encode": n * 2 + arc_bits_bytes,
        "K5_huff_decode": arc_bits_bytes + n * 2,
        "K6_reconstruct": n * 2 + 16 * n_out + n * s,
    }.get(name)


# ---------------------------------------------------------------------------
def cpu_oracle_run(values, dims, eb, threads):
    """One oracle compress + decompress; returns (t_compress, t_decompress, archive bytes)."""
    from oracle import oracle as O

    vmin, vmax = O.check_finite_minmax(values)
    t0 = time.perf_counter()
    arc = O.compress(values, dims, vmin, vmax, eb, threads=threads)
    t1 = time.perf_counter()
    O.decompress(arc, threads=threads)
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1, len(arc)


def _bits_at(data: "np.ndarray", bit_off: int, nbits: int):
    """nbits of an MSB-first byte stream starting at bit bit_off, re-aligned to
    bit 0 and zero padded to whole bytes (the layout of a standalone stream)."""
    import numpy as np

    lo = bit_off // 8
    hi = (bit_off + nbits + 7) // 8
    bits = np.unpackbits(np.asarray(data[lo: hi + 1], np.uint8))
    sh = bit_off - 8 * lo
    seg = bits[sh: sh + nbits]
    return np.packbits(seg).tobytes()


def parity_check(cfg, x, arc, ybuf, eb, threads):
    """Bit-exactness of the measured run against the CPU oracle, outside the
    timed region.

    Small configurations (C1-C4): the whole archive and the whole decoded
    field are compared with the oracle's.  C5-sized 3D fields (the oracle
    cannot hold 68 GB of int64 temporaries) are checked segment-wise:
      1. every 16-plane z-slab (two whole chunk layers, a contiguous range of
         the chunk-major stream and of the sorted outlier list) goes through
         the oracle's prequant + construct_stream with the GLOBAL eb_abs; the
         sum of the slab histograms must equal the device histogram, and the
         oracle's code book from it must equal the archive's;
      2. for sampled slabs (first, middle, last) the device code stream range,
         the archive's outlier records for that slab, the archive's bit stream
         at the slab's bit offset (oracle huff_encode of the slab stream with
         the global book) and the decoded slab (oracle reconstruct + dequant)
         must equal the oracle's, byte for byte."""
    import numpy as np
    import torch

    from oracle import oracle as O
    from paper_2105_12912_b200 import pipeline as PL

    t0 = time.perf_counter()
    hdr = arc.header
    shape = cfg["shape"]
    dims = dims_tuple(shape)
    n = x.numel()
    if n <= 400_000_000:
        xh = x.cpu().numpy()
        ref = O.compress(xh, dims, hdr.vmin, hdr.vmax, eb, threads=threads)
        got = arc.to_bytes()
        ok_arc = got == ref
        first = None
        if not ok_arc and len(got) == len(ref):
            first = int(np.flatnonzero(np.frombuffer(got, np.uint8) != np.frombuffer(ref, np.uint8))[0])
        want = O.decompress(ref, threads=threads)[0]
        ok_dec = bool(np.array_equal(ybuf[:n].cpu().numpy().view(np.uint8), want.view(np.uint8)))
        return {"ok": bool(ok_arc and ok_dec), "mode": "whole archive vs oracle",
                "archive_equal": bool(ok_arc), "first_diff_byte": first,
                "decode_equal": ok_dec, "oracle_threads": threads,
                "seconds": round(time.perf_counter() - t0, 1)}
    assert len(shape) == 3 and hdr.chunk.as_tuple() == (8, 8, 8)
    nz, ny, nx = shape
    plane = nx * ny
    P = 16
    nslab = nz // P
    cap, r = hdr.cap, hdr.cap // 2
    eb_abs = hdr.eb_abs
    sample = sorted({0, nslab // 2, nslab - 1})
    codes_dev = PL._pool.bufs[("codes", str(x.device))]
    hist_dev = PL._pool.bufs[("hist", str(x.device))][: cap * 8].cpu().numpy().view(np.int64)
    cb_off = hdr.codebook[0]
    lens_dev = arc.data[cb_off: cb_off + cap].cpu().numpy()
    out_off = hdr.outliers[0]
    rec_dev = arc.data[out_off: out_off + 16 * hdr.outlier_count].cpu().numpy().view(
        [("i", "<u8"), ("d", "<i8")])
    ghist = np.zeros(cap, np.int64)
    slab_hist = []
    kept = {}
    res = {"mode": "segment-wise (SURVEY 8(c) steps 1-3 + decoded slabs)", "slabs": nslab,
           "slab_planes": P, "sampled_slabs": sample, "oracle_threads": threads}
    ok = True
    for k in range(nslab):
        lo = k * P * plane
        xs = x[lo: lo + P * plane].cpu().numpy()
        pre = O.prequantize(xs, eb_abs, threads)
        stream, oi, od = O.construct_stream(pre, (nx, ny, P, 3), (8, 8, 8), r, threads)
        h = O.histogram(stream, cap)
        ghist += h
        slab_hist.append(h)
        if k in sample:
            dev_codes = codes_dev[2 * lo: 2 * (lo + P * plane)].cpu().numpy().view(np.uint16)
            c_ok = bool(np.array_equal(dev_codes, stream))
            a = np.searchsorted(rec_dev["i"], lo)
            b = np.searchsorted(rec_dev["i"], lo + P * plane)
            o_ok = bool(b - a == len(oi) and np.array_equal(rec_dev["i"][a:b] - lo, oi)
                        and np.array_equal(rec_dev["d"][a:b], od))
            kept[k] = (stream, oi, od, lo)
            res[f"slab{k}"] = {"codes_equal": c_ok, "outliers_equal": o_ok, "outliers": int(len(oi))}
            ok &= c_ok and o_ok
    h_ok = bool(np.array_equal(ghist, hist_dev))
    lens = O.huffman_lengths(ghist)
    b_ok = bool(np.array_equal(lens, lens_dev))
    res["histogram_equal"] = h_ok
    res["codebook_equal"] = b_ok
    ok &= h_ok and b_ok
    codes = O.canonical_codes(lens)
    L64 = lens.astype(np.int64)
    bit_before = np.cumsum([0] + [int((hh * L64).sum()) for hh in slab_hist])
    sym_off = hdr.symbols[0]
    for k, (stream, oi, od, lo) in kept.items():
        nb, _, data = O.huff_encode(stream, lens, codes)
        boff = int(bit_before[k])
        dlo = sym_off + 16 + boff // 8
        dhi = sym_off + 16 + (boff + nb + 7) // 8 + 1
        seg = arc.data[dlo: min(dhi, sym_off + hdr.symbols[1])].cpu().numpy()
        bits_ok = _bits_at(seg, boff % 8, nb) == data
        vals = O.reconstruct(stream, (nx, ny, P, 3), (8, 8, 8), r, oi, od, eb_abs, "f32", threads)
        d_ok = bool(np.array_equal(ybuf[lo: lo + P * plane].cpu().numpy().view(np.uint32),
                                   vals.view(np.uint32)))
        res[f"slab{k}"].update({"bit_offset": boff, "bits": nb, "bits_equal": bool(bits_ok),
                                "decode_equal": d_ok})
        ok &= bits_ok and d_ok
    res["ok"] = bool(ok)
    res["seconds"] = round(time.perf_counter() - t0, 1)
    return res


def sample_planes_for(cfg, target_elems):
    shape = cfg["shape"]
    per_plane = 1
    for s in shape[1:]:
        per_plane *= s
    return max(1, min(shape[0], target_elems // per_plane))


def dims_tuple(shape):
    ext = list(shape[::-1]) + [1] * (3 - len(shape))
    return (ext[0], ext[1], ext[2], len(shape))


def run_reference(args, cfg, rank, world):
    """--impl reference: the oracle port on all host threads, rank 0 only."""
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    planes = sample_planes_for(cfg, args.ref_sample_elems)
    vals, shp = gen_sample_host(cfg, planes)
    dims = dims_tuple(shp)
    nbytes = vals.nbytes
    for _ in range(args.warmup):
        cpu_oracle_run(vals, dims, cfg["eb"], threads)
    ts = []
    arc_len = 0
    for _ in range(args.steps):
        tc, td, arc_len = cpu_oracle_run(vals, dims, cfg["eb"], threads)
        ts.append((tc, td))
    t = statistics.mean(a + b for a, b in ts)
    val = nbytes / t / 1e9
    sample = f"{'x'.join(map(str, shp[::-1]))} sub-slab of {cfg['workload'].split(':')[0]} ({vals.size} elements)"
    line = {
        "impl": "reference", "metric": METRIC, "value": round(val, 6), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["workload"], "sample": sample, "threads": threads},
        "compress_gbs": round(nbytes / statistics.mean(a for a, _ in ts) / 1e9, 6),
        "decompress_gbs": round(nbytes / statistics.mean(b for _, b in ts) / 1e9, 6),
        "compression_ratio": round(nbytes / arc_len, 4),
        "cpu_baseline": {"value": round(val, 6), "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(val, 6), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_sharded(args, cfg, rank, world, dev, local_rank):
    """--gpus N (torchrun): strong scaling of the same field over N slabs of
    whole chunk layers.  A step is the round trip N=1 times:

      compress   = distributed.compress_sharded: histogram all-reduce,
                   (bits, outliers) all-gather, bit-phase encode -- every
                   rank ends holding its byte-exact slice of the archive;
      decompress = distributed.decompress_archive_sharded of the STORED
                   archive (every rank holds the whole archive, as after a
                   read): per-rank bit-range transfer maps, their
                   all-gather, range decode, all-to-all of the symbols to
                   the slab owners, slab reconstruct.

    The stored archive is built once, before timing, from the ranks' slices
    with one all-gather (distributed.allgather_archive) -- no rank
    compresses the full field.  Same metric as N=1: N*s / step time, each
    phase's time the max over ranks (CUDA events).  The slice-local
    decompress (a rank decoding the slice it just wrote, no exchange) is
    reported beside it as ``decompress_slice_local``."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2105_12912_b200 import ChunkSpec, Dims
    from paper_2105_12912_b200 import distributed as D

    shape = cfg["shape"]
    dims = Dims.of(*shape[::-1])
    chunk = ChunkSpec.default_for(dims.ndim)
    lo, hi = D.slab_bounds(dims, chunk, rank, world)
    x = gen_field_device(cfg, dev, lo, hi)
    mm = torch.stack([x.min().double(), -x.max().double()])  # global range (collective 0)
    dist.all_reduce(mm, op=dist.ReduceOp.MIN)
    vmin, vmax = float(mm[0]), float(-mm[1])
    ops = D.DeviceSlabOps(dev)
    eb = cfg["eb"]
    slack = float(np.spacing(np.float32(max(abs(vmin), abs(vmax))))) / 2
    bound = eb * (vmax - vmin) * (1 + 1e-12) + slack

    def compress(xin):
        return D.compress_sharded(ops, xin, dims, vmin, vmax, eb, "rel", 1024, chunk, 0)

    res = compress(x)
    arc = D.allgather_archive(res, device=dev)  # the stored archive, built once
    del res

    def step(xin):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record()
        res = compress(xin)
        e1.record()
        y, (alo, ahi), _ = D.decompress_archive_sharded(ops, arc)
        e2.record()
        assert (alo, ahi) == (lo, hi)
        return res, y, (e0, e1, e2)

    def max_over_ranks(vals):
        t = torch.tensor(vals, device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return [float(v) for v in t.cpu()]

    for _ in range(args.warmup):
        res, y, _ = step(x)
    torch.cuda.synchronize()
    ok = y is None or (y.double() - x.double()).abs().max().item() <= bound
    okt = torch.tensor([1 if ok else 0], device=dev, dtype=torch.int64)
    dist.all_reduce(okt, op=dist.ReduceOp.MIN)
    del y
    clocks = ClockSampler(local_rank)
    clocks.start()
    dist.barrier()
    torch.cuda.synchronize()
    clocks.mark("t0")
    tt, tc, td = [], [], []
    for _ in range(args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        res, y, (e0, e1, e2) = step(x)
        torch.cuda.synchronize()
        t = max_over_ranks([e0.elapsed_time(e2) / 1e3, e0.elapsed_time(e1) / 1e3,
                            e1.elapsed_time(e2) / 1e3])
        tt.append(t[0])
        tc.append(t[1])
        td.append(t[2])
        del y
    clocks.mark("t1")
    clk = clocks.stop()
    t_step, t_c, t_d = statistics.mean(tt), statistics.mean(tc), statistics.mean(td)

    # side number: each rank decodes the slice it just wrote (no exchange)
    tl = []
    for k in range(args.warmup + args.steps):
        dist.barrier()
        torch.cuda.synchronize()
        l0, l1 = (torch.cuda.Event(enable_timing=True) for _ in range(2))
        l0.record()
        yl = D.decompress_sharded(ops, res)
        l1.record()
        torch.cuda.synchronize()
        t = max_over_ranks([l0.elapsed_time(l1) / 1e3])[0]
        if k >= args.warmup:
            tl.append(t)
        ok_l = yl is None or (yl.double() - x.double()).abs().max().item() <= bound
        del yl
    okl = torch.tensor([1 if ok_l else 0], device=dev, dtype=torch.int64)
    dist.all_reduce(okl, op=dist.ReduceOp.MIN)

    n = dims.count
    nbytes = n * 4
    arc_bytes = int(arc.numel())
    # per GPU: its slab's algorithmic bytes (N*s + |archive| each way) over the step
    slab_bytes = (hi - lo) * (nbytes // shape[0])
    my_alg = 2 * (slab_bytes + arc_bytes * slab_bytes / nbytes)
    peak, peak_kind = measured_peak_hbm()
    ach = my_alg / t_step / 1e9

    # e2e: the slab from pinned host memory, its output back to the host.
    # The buffers are allocated first and every rank agrees before the timed
    # loop (a rank that failed to pin memory must not leave the others
    # waiting in a collective); a failure is reported in the line.
    e2e = None
    if args.e2e_steps > 0:
        bufs, err = None, None
        try:
            xh = torch.empty(x.numel(), dtype=x.dtype, pin_memory=True)
            xh.copy_(x)
            bufs = (xh, torch.empty_like(xh), torch.empty_like(x))
        except Exception as exc:  # pragma: no cover - box dependent
            err = repr(exc)[:300]
        okb = torch.tensor([1 if bufs is not None else 0], device=dev, dtype=torch.int64)
        dist.all_reduce(okb, op=dist.ReduceOp.MIN)
        if int(okb.item()) == 1:
            xh, yh, xd = bufs
            te = []
            for k in range(args.e2e_steps + 1):
                dist.barrier()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                xd.copy_(xh, non_blocking=True)
                res, y, _ = step(xd)
                yh.copy_(y, non_blocking=True)
                torch.cuda.synchronize()
                tk = max_over_ranks([time.perf_counter() - t0])[0]
                if k:
                    te.append(tk)
                del y
            v = statistics.mean(te)
            e2e = {"value": round(nbytes / v / 1e9, 4), "unit": "GB/s",
                   "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
                   "ms_per_step": round(v * 1e3, 2), "steps": args.e2e_steps,
                   "note": "per rank: its slab H2D, sharded compress + stored-archive decompress, "
                           "slab D2H; max over ranks"}
            del xh, yh, xd
        else:
            e2e = {"error": err or "another rank could not allocate its pinned buffers"}
        bufs = None
    if rank == 0:
        wf = res.meta["workflow"]
        print(json.dumps({
            "metric": METRIC, "value": round(nbytes / t_step / 1e9, 3), "unit": "GB/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(t_step * 1e3, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": cfg["workload"], "elements": n, "bytes": nbytes,
                       "workflow": wf, "parallelism": f"slab{world}",
                       "backend": dist.get_backend(),
                       "l2": "inputs >> 126 MB L2 (no flush)",
                       "step": "sharded compress (each rank ends with its byte-exact archive slice) + "
                               "decompress of the stored archive (range maps all-gather, range "
                               "decode, symbol all-to-all, slab reconstruct)"},
            "compress_gbs": round(nbytes / t_c / 1e9, 3), "decompress_gbs": round(nbytes / t_d / 1e9, 3),
            "compress_ms": round(t_c * 1e3, 3), "decompress_ms": round(t_d * 1e3, 3),
            "decompress_slice_local": {"decompress_gbs": round(nbytes / statistics.mean(tl) / 1e9, 3),
                                       "ms": round(statistics.mean(tl) * 1e3, 3),
                                       "bound_ok": bool(int(okl.item())),
                                       "what": "each rank decodes the slice it wrote (no exchange)"},
            "compression_ratio": round(nbytes / arc_bytes, 4), "archive_bytes": arc_bytes,
            "roofline": {"bound": "hbm", "kernel": "pipeline (per GPU, rank 0 slab)",
                         "achieved": round(ach, 1), "peak": peak, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": round(ach / peak, 4), "traffic": None},
            "bound_ok": bool(int(okt.item())),
            "gpu_launches": (LAUNCHES["lzb_quantize"] + LAUNCHES["lzb_codebook"] + LAUNCHES["lzb_huff_encode"]
                             + LAUNCHES["status_and_header_copies"]
                             + LAUNCHES["lzb_huff_decode"] + LAUNCHES["lzb_reconstruct_with_outliers"])
                            * args.steps * world,
            "clocks": clk, "e2e": e2e, "cpu_baseline": None,
        }), flush=True)


def run_gpu(args, cfg, rank, world, local_rank):
    import numpy as np
    import torch

    import paper_2105_12912_b200 as lzb
    from paper_2105_12912_b200 import _native

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    _native.lib()
    dist = None
    if world > 1:
        import torch.distributed as dist

    shape = cfg["shape"]
    if world > 1 or args.sharded:
        return run_sharded(args, cfg, rank, world, dev, local_rank)

    x = gen_field_device(cfg, dev)
    n = x.numel()
    s = x.element_size()
    field = lzb.Field.from_array(x.reshape(shape))
    eb = cfg["eb"]
    nbytes = n * s

    def step(prof=None, out=None):
        arc = lzb.compress_device(field, eb, prof=prof)
        y, hdr, _, _ = lzb.decompress_device(arc, prof=prof, out=out)
        return arc, y

    # field construction (reported separately): the device range
    # pass behind Field.from_array (lzb_field_range: min / max + first non-finite)
    fc = []
    for k in range(args.warmup + args.steps):
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        lzb.Field.from_array(x.reshape(shape))
        f1.record()
        torch.cuda.synchronize()
        if k >= args.warmup:
            fc.append(f0.elapsed_time(f1) / 1e3)
    t_fc = statistics.mean(fc)
    field_construction = {"ms": round(t_fc * 1e3, 3), "gbs": round(nbytes / t_fc / 1e9, 1),
                          "what": "Field.from_array of the device field: lzb_field_range "
                                  "(min / max / first non-finite), outside the step"}

    ybuf = torch.empty(n, dtype=x.dtype, device=dev)
    for _ in range(args.warmup):
        arc, y = step(out=ybuf)
    torch.cuda.synchronize()
    hdr = arc.header
    arc_len = arc.nbytes
    # correctness spot check of the warm-up output (bound + determinism)
    err = 0.0
    step_e = 1 << 28
    for a in range(0, n, step_e):
        err = max(err, (y[a:a + step_e].double() - x[a:a + step_e].double()).abs().max().item())
    slack = float(np.spacing(np.float32(max(abs(field.vmin), abs(field.vmax))))) / 2
    bound_ok = err <= hdr.eb_abs * (1 + 1e-12) + slack

    clocks = ClockSampler(local_rank)
    clocks.start()
    torch.cuda.synchronize()
    clocks.mark("t0")
    t_c, t_d, profs = [], [], []
    # inputs that fit in L2 (C1, C2): a 512 MB write evicts them before every timed step
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if nbytes < (512 << 20) else None
    # Stage events ride in the timed steps, except for fields small enough for
    # the single-sync compress: there they would serialise K2 with K1's outlier
    # compaction, so the stage times come from a second pass of the same steps.
    staged_in_timed = n > (1 << 25)
    for _ in range(args.steps):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        prof = [] if staged_in_timed else None
        if flush is not None:
            flush.zero_()
        e0.record()
        arc = lzb.compress_device(field, eb, prof=prof)
        e1.record()
        # the device API's round trip: decompress takes the DeviceArchive
        # compress returned (header known; no host read-back of the prefix)
        y, _, _, _ = lzb.decompress_device(arc, prof=prof, out=ybuf)
        e2.record()
        torch.cuda.synchronize()
        t_c.append(e0.elapsed_time(e1) / 1e3)
        t_d.append(e1.elapsed_time(e2) / 1e3)
        if prof is not None:
            profs.append(prof)
    torch.cuda.synchronize()
    clocks.mark("t1")
    clk = clocks.stop()
    if not staged_in_timed:
        for _ in range(args.steps):
            prof = []
            if flush is not None:
                flush.zero_()
            a = lzb.compress_device(field, eb, prof=prof)
            lzb.decompress_device(a, prof=prof, out=ybuf)
            torch.cuda.synchronize()
            profs.append(prof)
    tc, td = statistics.mean(t_c), statistics.mean(t_d)
    t_step = tc + td

    # per-stage device times (CUDA events on the launching stream)
    stage = {}
    for prof in profs:
        for name, a, b in prof:
            stage.setdefault(name, []).append(a.elapsed_time(b) / 1e3)
    stage_ms = {k: round(statistics.mean(v) * 1e3, 4) for k, v in stage.items()}
    bits_bytes = hdr.symbols[1] - 16 if hdr.workflow is lzb.Workflow.HUFFMAN else hdr.symbols[1]
    dom = max((k for k in stage if stage_bytes(k, n, s, bits_bytes, hdr.outlier_count)),
              key=lambda k: statistics.mean(stage[k]))
    peak, peak_kind = measured_peak_hbm()
    dom_bytes = stage_bytes(dom, n, s, bits_bytes, hdr.outlier_count)
    achieved = dom_bytes / statistics.mean(stage[dom]) / 1e9
    per_stage_roofline = {}
    for k in stage:
        b = stage_bytes(k, n, s, bits_bytes, hdr.outlier_count)
        if b:
            a = b / statistics.mean(stage[k]) / 1e9
            per_stage_roofline[k] = {"achieved_gbs": round(a, 1), "frac": round(a / peak, 4),
                                     "bytes": b}
    pipe_c = (nbytes + arc_len) / tc / 1e9
    pipe_d = (arc_len + nbytes) / td / 1e9

    # ---- bit-exactness of this run against the oracle (outside the timed region) ----
    parity = None
    if not args.no_parity:
        parity = parity_check(cfg, x, arc, ybuf, eb, os.cpu_count() or 1)

    # ---- e2e: host (pinned) buffers through the public device API ----
    # A stream of fields, pipelined the way a production loop would run it:
    # two device input buffers, so field k+2 uploads (copy engine, its own
    # stream) while field k is compressed, decompressed and downloaded (the
    # other copy engine; PCIe is full duplex).  The archive's trip to the host
    # and back is done by SM copy kernels over mapped pinned memory
    # (lzb_copy_bytes), so it does not queue behind the large DMA copies.
    # Every timed step still moves its whole field H2D, its archive D2H and
    # H2D and its whole result D2H inside the timed region; step 0 (warm-up)
    # runs alone and is finished before the clock starts.
    e2e = None
    if args.e2e_steps > 0:
        from paper_2105_12912_b200 import _native as N

        L = N.lib()
        xh = torch.empty(n, dtype=x.dtype, pin_memory=True)
        xh.copy_(x)
        dims, vmin, vmax = field.dims, field.vmin, field.vmax
        del field, x  # the device copy of the benchmark field is no longer needed
        torch.cuda.empty_cache()
        ah = torch.empty(arc_len + 4096, dtype=torch.uint8, pin_memory=True)
        yh = torch.empty(n, dtype=xh.dtype, pin_memory=True)
        xds = [torch.empty(n, dtype=xh.dtype, device=dev) for _ in range(2)]
        flds = [lzb.Field(dims, t, vmin, vmax) for t in xds]
        ad = torch.empty(arc_len + 4096, dtype=torch.uint8, device=dev)
        cs = torch.cuda.current_stream()
        up, down = torch.cuda.Stream(), torch.cuda.Stream()
        xready, xfree = [None, None], [None, None]
        state = {"yfree": None}
        trace = [] if os.environ.get("LZB_E2E_TRACE") else None

        def mark(stream, k, what):  # optional timeline (LZB_E2E_TRACE=1), off by default
            if trace is not None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(stream)
                trace.append((k, what, ev, time.perf_counter()))

        # The field upload of step k+2 and the result download of step k
        # share the host link in M chunk pairs: upload chunk j waits for
        # download chunk j-1.  Unpaced, the upload takes ~48 of the ~92 GB/s
        # duplex and finishes early while the download -- the critical path
        # (the next decompress waits for ybuf) -- crawls at ~36 GB/s.
        M = 8
        bounds = [n * j // M for j in range(M + 1)]
        dn_events = {}

        def upload(k):
            b = k % 2
            pace = dn_events.get(k - 2)
            with torch.cuda.stream(up):
                if xfree[b] is not None:
                    up.wait_event(xfree[b])  # the compress that read this buffer is done
                mark(up, k, "up0")
                for j in range(M):
                    if pace is not None and j > 0:  # chunk 0 goes at once; then one behind the download
                        up.wait_event(pace[j - 1])
                    xds[b][bounds[j]: bounds[j + 1]].copy_(xh[bounds[j]: bounds[j + 1]], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(up)
                xready[b] = ev
                mark(up, k, "up1")

        def one_step(k, last):
            b = k % 2
            cs.wait_event(xready[b])
            mark(cs, k, "c0")
            a = lzb.compress_device(flds[b], eb)  # returns after its status read
            mark(cs, k, "c1")
            ev = torch.cuda.Event()
            ev.record(cs)
            xfree[b] = ev
            sp = N.stream_ptr()
            N.check_rc(L.lzb_copy_bytes(ah.data_ptr(), a.data.data_ptr(), a.nbytes, sp), "copy")  # D2H
            N.check_rc(L.lzb_copy_bytes(ad.data_ptr(), ah.data_ptr(), a.nbytes, sp), "copy")      # H2D
            mark(cs, k, "arc")
            cs.synchronize()  # the host copy of the archive is complete
            pre = ah[: a.header.symbols[0] + 32].numpy().tobytes()
            if state["yfree"] is not None:
                cs.wait_event(state["yfree"])  # the previous result has left ybuf
            mark(cs, k, "d0")
            yy, _, _, _ = lzb.decompress_device(ad[: a.nbytes], raw_host=pre, out=ybuf)
            done = torch.cuda.Event()
            done.record(cs)
            mark(cs, k, "d1")
            with torch.cuda.stream(down):
                down.wait_event(done)
                mark(down, k, "dn0")
                evs = []
                for j in range(M):
                    yh[bounds[j]: bounds[j + 1]].copy_(yy[bounds[j]: bounds[j + 1]], non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(down)
                    evs.append(e)
                dn_events[k] = evs
                dn_events.pop(k - 3, None)
                yf = evs[-1]
                mark(down, k, "dn1")
            state["yfree"] = yf
            if k + 2 <= last:
                upload(k + 2)  # paced by this step's download chunks

        upload(0)
        one_step(0, 0)  # warm-up: pinned paths, pools
        torch.cuda.synchronize()
        ok_e2e = bool(torch.equal(yh[:1 << 20].to(dev), ybuf[:1 << 20]))
        # slices of the finished step-0 result: every timed step decodes the same
        # field, so the LAST timed step's downloaded result must match them
        probe = [0, n // 2 - (1 << 19), n - (1 << 20)] if n > (1 << 21) else [0]
        pw = min(n, 1 << 20)
        ref_sl = [ybuf[a: a + pw].clone() for a in probe]
        K = args.e2e_steps
        t0 = time.perf_counter()
        upload(1)
        if K >= 2:
            upload(2)
        for k in range(1, K + 1):
            one_step(k, K)
        down.synchronize()
        torch.cuda.synchronize()
        te = (time.perf_counter() - t0) / K
        if trace:
            base = next(ev for kk, w, ev, _ in trace if kk == 1 and w == "up0")
            for kk, w, ev, th in trace:
                if kk >= 1:
                    print(f"e2e-trace step {kk:2d} {w:4s} gpu {base.elapsed_time(ev):9.1f} ms "
                          f"host {1e3 * (th - t0):9.1f} ms", file=sys.stderr)
        ok_e2e = ok_e2e and all(bool(torch.equal(yh[a: a + pw].to(dev), rs))
                                for a, rs in zip(probe, ref_sl))
        e2e = {"value": round(nbytes / te / 1e9, 4), "unit": "GB/s",
               "h2d_bytes_per_step": nbytes + arc_len, "d2h_bytes_per_step": arc_len + nbytes,
               "ms_per_step": round(te * 1e3, 2), "steps": K,
               "pipelined": "field uploads run two steps ahead (two device input buffers), paced "
                            "chunk by chunk against the result download they share the link with; "
                            "archive copies by SM kernels beside the DMA transfers",
               "result_check": ok_e2e,
               "result_check_what": "last timed step's downloaded field == step-0 result at 3 slices"}
        del xh, ah, yh, xds, flds, ad

    # ---- CPU baseline: oracle port, 1 thread, bounded sub-slab ----
    cpu = None
    if not args.no_cpu_baseline:
        planes = sample_planes_for(cfg, args.cpu_sample_elems)
        vals, shp = gen_sample_host(cfg, planes)
        tc0, td0, alen = cpu_oracle_run(vals, dims_tuple(shp), eb, 1)
        cpu = {"value": round(vals.nbytes / (tc0 + td0) / 1e9, 6), "unit": "GB/s", "cores": 1,
               "kind": "port",
               "sample": f"{'x'.join(map(str, shp[::-1]))} sub-slab of the workload "
                         f"({vals.size} elements), compress {tc0:.2f}s + decompress {td0:.2f}s"}

    line = {
        "metric": METRIC, "value": round(nbytes / t_step / 1e9, 3), "unit": "GB/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(t_step * 1e3, 3), "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["workload"], "elements": n, "bytes": nbytes,
                   "workflow": hdr.workflow.name,
                   "l2": "inputs >> 126 MB L2 (no flush)" if nbytes >= (512 << 20) else
                         "L2 flushed (512 MB write) before every timed step",
                   "decompress_input": "the DeviceArchive compress_device returned",
                   "parallelism": f"slab{world}" if world > 1 else "single"},
        "compress_gbs": round(nbytes / tc / 1e9, 3),
        "decompress_gbs": round(nbytes / td / 1e9, 3),
        "compress_ms": round(tc * 1e3, 3), "decompress_ms": round(td * 1e3, 3),
        "compression_ratio": round(nbytes / arc_len, 4), "archive_bytes": arc_len,
        "outliers": hdr.outlier_count,
        "pipeline_roofline": {"compress_frac": round(pipe_c / peak, 4),
                              "decompress_frac": round(pipe_d / peak, 4),
                              "compress_gbs_alg": round(pipe_c, 1),
                              "decompress_gbs_alg": round(pipe_d, 1),
                              "bytes": "N*4 + |archive| per direction (SURVEY 8(d))"},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1),
                     "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": round(achieved / peak, 4), "traffic": profiled_traffic(dom),
                     "traffic_source": "profiles/ncu_traffic.json: ncu dram__bytes_read+write of this "
                                       "stage's kernels in one step of this command (tools/launch_summary.py)"},
        "stages_ms": stage_ms, "stage_roofline": per_stage_roofline,
        "bound_ok": bool(bound_ok), "max_abs_err": err, "eb_abs": hdr.eb_abs,
        "gpu_launches": launches_per_step(hdr) * args.steps,
        "clocks": clk, "e2e": e2e, "cpu_baseline": cpu, "parity": parity,
        "field_construction": field_construction,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lzb", choices=["lzb", "reference"])
    ap.add_argument("--config", default="c5", choices=sorted(CONFIGS))
    ap.add_argument("--e2e-steps", type=int, default=16)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-parity", action="store_true",
                    help="skip the post-run oracle comparison (profiling runs)")
    ap.add_argument("--cpu-sample-elems", type=int, default=2048 * 2048 * 32)
    ap.add_argument("--ref-sample-elems", type=int, default=2048 * 2048 * 16)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N>1 (gloo only for one-GPU debugging)")
    ap.add_argument("--sharded", action="store_true",
                    help="check: run the N>1 slab path (process group, NCCL collectives) even at N=1")
    ap.add_argument("--same-device", action="store_true",
                    help="debug: put every rank on cuda:0 (with --backend gloo)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = CONFIGS[args.config]
    use_pg = world > 1 or (args.sharded and args.impl != "reference")
    if use_pg:
        import torch
        import torch.distributed as dist

        backend = "gloo" if args.impl == "reference" else args.backend
        if args.same_device:  # debug: every rank on cuda:0 (one-GPU check of the N>1 path)
            local_rank = 0
        if args.impl != "reference":
            torch.cuda.set_device(local_rank)
        dist.init_process_group(backend)
    try:
        if args.impl == "reference":
            run_reference(args, cfg, rank, world)
        else:
            run_gpu(args, cfg, rank, world, local_rank)
    finally:
        if use_pg:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
