#!/usr/bin/env python
"""SZx compress/decompress throughput on B200 (BASELINE.json metric).

Workload at N=1: BASELINE.json configs[1], the NYX-shaped 512^3 float32 field
(smooth-ridges synthetic data generated on the device), value-range-relative eb 1e-3 as the
headline (the 1e-2 / 1e-4 legs of the sweep are reported beside it), block size 128.

A step = one compress (K1, which also writes the decode index as a by-product of its
look-back) + one decompress (K2 decoding through that index) of the whole field with inputs
resident in HBM; value = 2 * field bytes / (compress + decompress device time), i.e. GB/s of
field data through the codec in both directions.  A stream that arrives as bytes needs the
index pass K3 before K2; it is timed separately (roofline.per_kernel.index128_kernel,
roofline.step_ms.decompress_from_bytes_k3_plus_k2) and is part of every e2e decompress.  e2e = the same through the C-ABI host-buffer
entry points (szx_compress_host / szx_decompress_host) from/to pinned host memory.

Multi-GPU (torchrun, N>1): each rank owns a block-aligned shard of an N-times-larger field
(weak scaling); NCCL all-reduces the range once (rel bound) and all-gathers the per-shard
pool totals every step -- the exchange a single-stream assembly needs.

--impl reference: the reference's algorithm on the host cores (the C restatement in
oracle/, multithreaded over block-aligned shards), rank 0 only.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SZx compress/decompress GB/s at 1/2/4/8 B200 vs HBM roofline; compression ratio"
UNIT = "GB/s"
CONFIGS = {
    "nyx": {"dims": (512, 512, 512), "kind": "smooth_ridges",
            "name": "NYX-shaped 512^3 float32 smooth_ridges (BASELINE configs[1])"},
    "hurricane": {"dims": (100, 500, 500), "kind": "smooth_ridges",
                  "name": "Hurricane-ISABEL-shaped 100x500x500 float32 smooth_ridges (configs[0])"},
    "hacc": {"dims": (280_953_867,), "kind": "random_walk",
             "name": "HACC-shaped 280,953,867 float32 random_walk (configs[3])"},
    "hacc_ridges": {"dims": (280_953_867,), "kind": "smooth_ridges",
                    "name": "HACC-shaped 280,953,867 float32 smooth_ridges (configs[3], 2nd "
                            "generator)"},
    "shard": {"dims": (24_414_080 * 128,), "kind": "smooth_ridges",
              "name": "one 12.5 GB shard (3,125,002,240 float32 smooth_ridges) of the ~100 GB "
                      "field: the per-GPU work of BASELINE configs[4]"},
    "cesm": {"dims": (1800, 3600), "kind": "smooth_ridges", "fields": 77,
             "name": "CESM-ATM-shaped 77 x 1800x3600 float32 smooth_ridges, rel bound per "
                     "field (BASELINE configs[2]), batched"},
}
L2_BYTES = 126 * 1024 * 1024


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", float(
            p.get("sm_max_mhz", 1965))
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)", 1965.0


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling through NVML during timed work."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, index: int):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        self._t = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# --------------------------------------------------------------------------------------
# CPU baseline: the oracle (reference algorithm restated in C), all host threads
# --------------------------------------------------------------------------------------
class OracleRunner:
    def __init__(self, n: int, bs: int = 128, ndims: int = 3):
        import oracle

        self.ndims = ndims
        self.o = oracle
        self.L = oracle.lib()
        self.n, self.bs = n, bs
        nb = -(-n // bs)
        self.map = np.zeros((nb + 7) // 8 + 8, np.uint8)
        self.mu = np.zeros(nb + 4, np.float32)
        self.req = np.zeros(nb + 8, np.uint8)
        self.codes = np.zeros(n // 4 + 8, np.uint8)
        self.mid = np.zeros(4 * n + 8, np.uint8)
        self.out = np.zeros(n, np.float32)
        for a in (self.map, self.mu, self.req, self.codes, self.mid, self.out):
            a.fill(1)  # fault the pages in before timing

    def run(self, x: np.ndarray, e: float, threads: int):
        P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
        sz = self.o._Sizes()
        t0 = time.perf_counter()
        rc = self.L.szxo_compress_mt(P(x), x.size, self.bs, e, threads, P(self.map), P(self.mu),
                                     P(self.req), P(self.codes), P(self.mid), ctypes.byref(sz))
        t1 = time.perf_counter()
        assert rc == 0
        rc = self.L.szxo_decompress_mt(P(self.map), P(self.mu), P(self.req), P(self.codes),
                                       P(self.mid), sz.mid_len, x.size, self.bs, threads,
                                       P(self.out))
        t2 = time.perf_counter()
        assert rc == 0
        nb = -(-x.size // self.bs)
        c = 17 + 8 * self.ndims + (nb + 7) // 8 + 4 * nb + sz.n_nc + (2 * sz.m + 7) // 8 + sz.mid_len
        return t1 - t0, t2 - t1, c


def stream_parity(s, x, out) -> str:
    """tests/streamcheck.check_stream on the bench's own stream (checker only, after timing)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from streamcheck import check_stream

    st = check_stream(s, x, out, window_blocks=1 << 20)
    return f"bit-exact vs oracle ({st['windows']} windows, every pool byte + reconstruction)"


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def cpu_baseline(x_host: np.ndarray, e: float, budget_s: float = 12.0):
    """Time the oracle port on a bounded leading sample of the workload."""
    threads = cpu_cores()
    r = OracleRunner(x_host.size)
    tc, td, c = r.run(x_host, e, threads)  # warm-up
    reps = max(1, min(20, int(budget_s / max(tc + td, 1e-3))))
    best_c, best_d = [], []
    for _ in range(reps):
        tc, td, c = r.run(x_host, e, threads)
        best_c.append(tc)
        best_d.append(td)
    tc, td = statistics.median(best_c), statistics.median(best_d)
    nbytes = 4 * x_host.size
    return {
        "value": round(2 * nbytes / (tc + td) / 1e9, 4),
        "unit": UNIT,
        "cores": threads,
        "kind": "port",
        "sample": f"first {x_host.size:,} values ({nbytes / 2**20:.0f} MiB) of the workload, "
                  f"bs 128, same abs bound; compress+decompress, median of {reps}; "
                  f"oracle/szx_oracle.c over {threads} threads on {cpu_model()}",
        "compress_gbs": round(nbytes / tc / 1e9, 4),
        "decompress_gbs": round(nbytes / td / 1e9, 4),
    }


# --------------------------------------------------------------------------------------
# distributed helpers
# --------------------------------------------------------------------------------------
def host_launches(L, n: int, bs: int) -> int:
    """Kernels one szx_compress_host + szx_decompress_host round trip launches (fast block
    sizes): K0, one K1 per launch chunk (<= 2^26 - 64 blocks), then K3 over the first decode
    chunk's pool prefixes, K3, the chunk-plan kernel and one K2 per decode chunk."""
    parts = int(L.szx_set_host_pipeline(0, 0))  # 0: query (the part count stays)
    nb = -(-n // bs)
    cap = ((1 << 26) - 64) // 64 * 64
    ntiles = -(-n // 8192)
    chunks = sum(1 for j in range(parts) if ntiles * (j + 1) // parts > ntiles * j // parts)
    prefix = 1 if parts >= 2 and ntiles // parts >= 1 else 0
    return 1 + -(-nb // cap) + prefix + 1 + 1 + chunks


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="nyx", choices=sorted(CONFIGS))
    ap.add_argument("--rel", type=float, default=1e-3)
    ap.add_argument("--sweep", default="1e-2,1e-4", help="extra rel bounds reported beside")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--cpu-sample", type=int, default=1 << 24,
                    help="values of the cpu_baseline leg of our arm (a bounded sample)")
    ap.add_argument("--ref-sample", type=int, default=0,
                    help="values timed by --impl reference (0: the whole workload field)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--kernel-reps", type=int, default=20,
                    help="per-kernel timing repetitions (K1, K3, K2 separately)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3

    ws, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, ws, rank)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return self_launch(args.gpus)
    if ws != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws}", file=sys.stderr)
        return 2
    if args.config == "cesm":
        return run_cesm(args, ws, rank, local)
    return run_ours(args, ws, rank, local)


def self_launch(ngpus: int) -> int:
    """`bench.py --gpus N` outside torchrun: start N ranks (one per GPU) under
    torch.distributed.run on this node; fail loudly when the node has fewer GPUs."""
    import socket
    import subprocess

    import torch

    have = torch.cuda.device_count()
    if have < ngpus:
        print(f"bench.py: --gpus {ngpus} needs {ngpus} GPUs, this node has {have}",
              file=sys.stderr)
        return 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={ngpus}", "--master-addr=127.0.0.1", f"--master-port={port}",
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_cesm(args, ws, rank, local):
    """BASELINE configs[2]: 77 CESM-shaped fields per GPU, each with its own relative bound,
    through the batched path -- ONE K1 launch over all fields' tiles (compress), ONE K3 + ONE
    K2 launch (decompress).  Step = batched compress + batched decompress, device events;
    value = 2 * field bytes / step time.  e2e = the user-level batch API from pinned host
    tensors: datafields + compress_batch + serialize, deserialize + decompress_batch + .values."""
    import torch

    import paper_2201_13020_b200 as szx
    from paper_2201_13020_b200 import synth

    torch.cuda.set_device(local)
    if ws > 1:
        print("bench.py --config cesm: one GPU per run (the batch is a per-GPU workload)",
              file=sys.stderr)
        return 2
    cfg = CONFIGS["cesm"]
    dims, nf = cfg["dims"], cfg["fields"]
    n = int(np.prod(dims))
    hbm_peak, peak_src, _ = peaks()
    xs = [synth.field("smooth_ridges", n, seed=i) for i in range(nf)]
    ccfg = szx.CompressorConfig(szx.ErrorBound("rel", args.rel))
    fs = szx.datafields(xs, [dims] * nf)
    stream = torch.cuda.current_stream()
    sp = int(stream.cuda_stream)
    st = szx.compress_batch(fs, ccfg)  # the streams (and the arena they live in)
    outs = szx.decompress_batch(st)
    # the timed launches: the batched ABI calls themselves on pre-built argument arrays
    # (what compress_batch / decompress_batch issue), back to back without host syncs
    from paper_2201_13020_b200 import _abi, _device

    L = _abi.lib()
    P = _device.ptr
    vp, u64 = ctypes.c_void_p, ctypes.c_uint64
    arr = lambda t, vals: (t * nf)(*vals)  # noqa: E731
    ns = arr(u64, [n] * nf)
    pools = [s.device_pools for s in st]
    c_args = (nf, arr(vp, [P(f.device_values) for f in fs]), ns,
              arr(ctypes.c_double, [s.error_bound for s in st]),
              arr(vp, [P(s._map) for s in st]), arr(vp, [P(s._mu) for s in st]),
              arr(vp, [P(s._req) for s in st]), arr(vp, [P(s._codes) for s in st]),
              arr(vp, [P(s._mid_buf) for s in st]))
    totals = torch.zeros(4 * nf, dtype=torch.int64, device="cuda")
    cerr = torch.zeros(2, dtype=torch.int64, device="cuda")
    csc = _device.empty_u8(L.szx_compress_batch_scratch_bytes(nf, ns))
    d_args = (nf, arr(vp, [P(p["constant_map"]) for p in pools]), arr(vp, [P(p["mu"]) for p in pools]),
              arr(vp, [P(s._req) for s in st]), arr(vp, [P(s._codes) for s in st]),
              arr(vp, [P(s._mid_buf) for s in st]), arr(u64, [s.mid_len for s in st]), ns,
              arr(vp, [P(o.device_values) for o in outs]))
    derr = torch.zeros(nf, dtype=torch.int32, device="cuda")
    dsc = _device.empty_u8(L.szx_decompress_batch_scratch_bytes(nf, ns))
    idx_args = arr(vp, [P(s._index) for s in st])  # the decode indexes compress_batch wrote

    def k_compress():  # K1 over all fields + the decode-index entries from its group offsets
        assert L.szx_compress_batch_indexed_f32(*c_args, idx_args, P(totals), P(cerr), P(csc),
                                                csc.numel(), sp) == 0

    def k_decompress():  # K2 over all fields' decode tiles through those indexes
        assert L.szx_decompress_batch_indexed_f32(*d_args[:-1], idx_args, d_args[-1], P(derr),
                                                  P(dsc), dsc.numel(), sp) == 0

    for _ in range(args.warmup):
        k_compress()
        k_decompress()
    torch.cuda.synchronize()
    N4 = 4 * n * nf
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        for k in range(args.steps):  # (inputs: 1.9 GiB > L2, no flush needed)
            ev[k][0].record(stream)
            k_compress()
            ev[k][1].record(stream)
            ev[k][2].record(stream)
            k_decompress()
            ev[k][3].record(stream)
        torch.cuda.synchronize()
    tc = [ev[k][0].elapsed_time(ev[k][1]) for k in range(args.steps)]
    td = [ev[k][2].elapsed_time(ev[k][3]) for k in range(args.steps)]
    tc_ms, td_ms = statistics.median(tc), statistics.median(td)
    assert int(cerr[0].item()) == 0 and int(derr.abs().sum().item()) == 0
    # the timed launches rewrote the same pools / outputs: they are what is checked below
    h = totals.cpu().numpy().reshape(-1, 4)
    assert all(int(h[i, 2]) == s.mid_len and int(h[i, 0]) == s._n_nc for i, s in enumerate(st))
    C = sum(s.compressed_size_bytes() for s in st)
    # parity on the timed data: every field's stream bytes and reconstruction bits vs the
    # oracle (the reference algorithm in C)
    import oracle

    bad = 0
    for i, (x, s, o) in enumerate(zip(xs, st, outs)):
        xh = x.cpu().numpy()
        ref = oracle.compress(xh, dims, 128, "rel", args.rel, nthreads=cpu_cores())
        bad += szx.serialize(s) != ref
        bad += not np.array_equal(o.device_values.cpu().numpy().view(np.uint32),
                                  oracle.decompress(ref, nthreads=cpu_cores()).view(np.uint32))
    assert bad == 0, f"{bad} CESM fields differ from the oracle"
    err = max(float((x.double() - o.device_values.double()).abs().max()) / s.error_bound
              for x, s, o in zip(xs, st, outs))
    # e2e through the public batch API from pinned host tensors
    hx = [x.cpu().pin_memory() for x in xs]
    e2e_t = []
    for k in range(max(args.e2e_steps, 1) + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        blobs = [szx.serialize(s) for s in szx.compress_batch(szx.datafields(hx, [dims] * nf),
                                                              ccfg)]
        vals = [o.values for o in szx.decompress_batch([szx.deserialize(b) for b in blobs])]
        t1 = time.perf_counter()
        if k:
            e2e_t.append(t1 - t0)
    te = statistics.median(e2e_t)
    assert all(np.array_equal(v, o.device_values.cpu().numpy()) for v, o in zip(vals[:2], outs))
    line = {
        "metric": METRIC, "value": round(2 * N4 / ((tc_ms + td_ms) * 1e-3) / 1e9, 3),
        "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(tc_ms + td_ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["name"], "fields": nf, "dims": list(dims), "rel_eb": args.rel,
                   "block_size": 128, "parallelism": "single",
                   "l2": f"input {N4 / 2**30:.2f} GiB > L2 (no flush)",
                   "step": "compress_batch (one K1 launch + the decode-index entries) + "
                           "decompress_batch (one K2 launch through those indexes), device "
                           "events (median)"},
        "compress_gbs": round(N4 / (tc_ms * 1e-3) / 1e9, 3),
        "decompress_gbs": round(N4 / (td_ms * 1e-3) / 1e9, 3),
        "cr": round(N4 / C, 4), "compressed_bytes": C,
        "max_abs_err_over_eb": round(err, 6),
        "parity": f"bit-exact vs oracle: all {nf} fields' streams and reconstructions",
        "roofline": {"bound": "hbm", "kernel": "compress128v3_kernel<batch>",
                     "achieved": round((N4 + C) / (tc_ms * 1e-3) / 1e9, 2), "peak": hbm_peak,
                     "unit": "GB/s",
                     "frac": round((N4 + C) / (tc_ms * 1e-3) / 1e9 / hbm_peak, 4),
                     "traffic": None, "peak_source": peak_src,
                     "algorithmic_bytes": N4 + C,
                     "decode_frac": round((N4 + C) / (td_ms * 1e-3) / 1e9 / hbm_peak, 4)},
        "e2e": {"value": round(2 * N4 / te / 1e9, 3), "unit": UNIT,
                "h2d_bytes_per_step": N4 + C, "d2h_bytes_per_step": C + N4,
                "ms_per_step": round(1e3 * te, 2),
                "path": "datafields(pinned host tensors) + compress_batch + serialize; "
                        "deserialize + decompress_batch + .values"},
        # timed step: K1 + index entries + K2 (batched); each e2e step: the batched K0, K1 and
        # index entries, then per field the validate pass and K3 of deserialize, then the
        # batched K2 (through deserialize's indexes)
        "gpu_launches": 3 * args.steps + (2 * nf + 4) * len(e2e_t),
        "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    return 0


def run_reference(args, ws, rank):
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import fields as fields_host  # the reference generators restated (tests/fields.py)

    cfg = CONFIGS[args.config]
    nfields = cfg.get("fields", 1)
    if nfields > 1:  # CESM: --ref-sample = fields timed (default: all of them)
        nfields = min(args.ref_sample, nfields) if args.ref_sample > 0 else nfields
        full = n = int(np.prod(cfg["dims"]))
        xs = [fields_host.smooth_ridges(np.random.default_rng(i), n) for i in range(nfields)]
    else:
        full = int(np.prod(cfg["dims"]))
        n = min(args.ref_sample, full) if args.ref_sample > 0 else full
        rng = np.random.default_rng(0)
        xs = [fields_host.smooth_ridges(rng, n) if cfg["kind"] == "smooth_ridges"
              else fields_host.random_walk(rng, n, step=0.01)]
    es = [args.rel * (float(x.max()) - float(x.min())) for x in xs]
    threads = cpu_cores()
    r = OracleRunner(n, ndims=len(cfg["dims"]))
    for _ in range(args.warmup):
        r.run(xs[0], es[0], threads)
    tcs, tds, c = [], [], 0
    for _ in range(args.steps):
        c = 0
        for x, e in zip(xs, es):
            tc, td, ci = r.run(x, e, threads)
            tcs.append(tc)
            tds.append(td)
            c += ci
    n = n * len(xs)
    t = sum(tcs) + sum(tds)
    value = 2 * 4 * n * args.steps / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * t / args.steps, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["name"] + (f" -- host sample of {n:,} values" if n < full * cfg.get("fields", 1)
                                              else " -- the whole workload, host-resident"),
                   "dims": list(cfg["dims"]), "rel_eb": args.rel, "block_size": 128,
                   "n_values": n, "same_config": n == full * cfg.get("fields", 1),
                   "l2": "host-resident field (no device)"},
        "compress_gbs": round(4 * n * args.steps / sum(tcs) / 1e9, 4),
        "decompress_gbs": round(4 * n * args.steps / sum(tds) / 1e9, 4),
        "cr": round(4 * n / c, 4),
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": threads,
                         "kind": "port",
                         "sample": f"{n:,} values ({'the whole field' if n == full else 'sample'}"
                                   f") {cfg['kind']}(seed 0) generated on the host with the "
                                   f"reference generator restatement (tests/fields.py == "
                                   f"ufzx/synth.py); oracle/szx_oracle.c (the reference "
                                   f"algorithm in C) over {threads} threads, block-aligned "
                                   f"shards, on {cpu_model()}"},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def run_ours(args, ws, rank, local):
    import torch

    import paper_2201_13020_b200 as szx
    from paper_2201_13020_b200 import _abi, _device, synth
    from paper_2201_13020_b200.pipeline import (_Pools, compress_device, decompress_device,
                                                index_buffer)

    torch.cuda.set_device(local)
    dist = None
    if ws > 1:
        import torch.distributed as dist

        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = CONFIGS[args.config]
    dims = cfg["dims"]
    n = int(np.prod(dims))
    bs = 128
    hbm_peak, peak_src, sm_max = peaks()
    L = _abi.lib()

    # field: each rank owns one NYX-sized, block-aligned shard of a ws-times-larger field
    x = synth.field(cfg["kind"], n, seed=1000 + rank)
    torch.cuda.synchronize()
    mm = torch.stack([x.min(), x.max()])
    if dist is not None:  # rel bound over the GLOBAL range (the one NCCL all-reduce)
        lo, hi = mm[0:1].clone(), mm[1:2].clone()
        dist.all_reduce(lo, op=dist.ReduceOp.MIN)
        dist.all_reduce(hi, op=dist.ReduceOp.MAX)
        mm = torch.cat([lo, hi])
    gmin, gmax = (float(v) for v in mm.cpu())
    stream = torch.cuda.current_stream()
    sp = int(stream.cuda_stream)

    results = {}
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.float32, device="cuda")
    for rel in [args.rel] + [float(v) for v in args.sweep.split(",") if v]:
        e = rel * (gmax - gmin)
        pools = _Pools(n, bs)
        small = torch.zeros(8, dtype=torch.int64, device="cuda")
        out = torch.empty(n, dtype=torch.float32, device="cuda")
        dsmall = torch.zeros(8, dtype=torch.int64, device="cuda")
        dscratch = _device.Scratch.get("decompress", L.szx_decompress_scratch_bytes(n, bs))
        tot_all = torch.zeros(4 * ws, dtype=torch.int64, device="cuda")
        mid_all = torch.zeros(ws, dtype=torch.int64, device="cuda")

        # K1 also writes the decode index (szx_compress_indexed_f32), which the decode of
        # this device-produced stream uses instead of running K3 (a deserialized stream's
        # decode runs K3: timed separately below as index128_kernel)
        idx = index_buffer(n, bs)

        def one_compress():
            compress_device(x, n, bs, e, pools, small, sp, idx)

        # stream object for decode (built once from the first compress)
        one_compress()
        h = small.cpu().numpy()
        s = szx.CompressedStream._from_device(
            bs, e, dims, pools.map, pools.mu[: 4 * (-(-n // bs))].view(torch.float32), pools.req,
            pools.codes, pools.mid, int(h[0]), int(h[1]), int(h[2]))
        s._index = idx
        assert int(h[4]) == 0

        def one_decompress():
            decompress_device(s, out, dsmall, dscratch, sp)

        for _ in range(args.warmup):
            one_compress()
            one_decompress()
        torch.cuda.synchronize()
        # correctness guard on the timed data: bound holds, stream deterministic
        err = float((x.double() - out.double()).abs().max())
        assert err <= e, (err, e)
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(4)] for _ in range(args.steps)]
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        t_start = time.perf_counter()
        with ClockSampler(local) as clk:
            for k in range(args.steps):
                flush.zero_()  # L2 flush between timed kernels (outside the events)
                ev[k][0].record(stream)
                one_compress()
                if dist is not None:  # per-shard totals -> stream offsets (NCCL all-gather)
                    dist.all_gather_into_tensor(tot_all, small[:4])
                ev[k][1].record(stream)
                flush.zero_()
                ev[k][2].record(stream)
                one_decompress()
                if dist is not None:  # shard mid totals -> mid-pool offsets (sharded decode)
                    dist.all_gather_into_tensor(mid_all, small[2:3])
                ev[k][3].record(stream)
            torch.cuda.synchronize()
        wall = time.perf_counter() - t_start
        tc = [ev[k][0].elapsed_time(ev[k][1]) for k in range(args.steps)]
        td = [ev[k][2].elapsed_time(ev[k][3]) for k in range(args.steps)]
        tsum = torch.tensor([sum(tc), sum(td)], dtype=torch.float64, device="cuda")
        if dist is not None:
            dist.all_reduce(tsum, op=dist.ReduceOp.MAX)
        tc_ms, td_ms = (float(v) / args.steps for v in tsum.cpu())
        h = small.cpu().numpy()
        n_nc, m, mid_len = int(h[0]), int(h[1]), int(h[2])
        nb = -(-n // bs)
        c_bytes = 17 + 8 * len(dims) + -(-nb // 8) + 4 * nb + n_nc + -(-2 * m // 8) + mid_len
        results[rel] = {"tc_ms": tc_ms, "td_ms": td_ms, "c": c_bytes, "err": err, "e": e,
                        "n_nc": n_nc, "m": m,
                        "clocks": clk.summary(), "wall_s": wall, "pools": pools, "stream": s}
        # parity on the timed data: every pool byte and every reconstructed value against the
        # oracle (the reference algorithm in C), window by window over the whole field
        results[rel]["parity"] = stream_parity(s, x, out)
        if rel != args.rel:
            del pools, s
            results[rel].pop("pools")
            results[rel].pop("stream")

    head = results[args.rel]
    N4 = 4 * n

    # ---- per-kernel device times of the headline leg (K3 index and K2 decode separately) --
    kt = {}
    if args.kernel_reps > 0:
        pools, s = head["pools"], head["stream"]
        nbk = -(-n // bs)
        p = s.device_pools
        idx3 = torch.empty(L.szx_index_bytes(n, bs) // 8, dtype=torch.int64, device="cuda")
        isc = _device.empty_u8(L.szx_index_scratch_bytes(n, bs))
        st4 = torch.zeros(4, dtype=torch.int64, device="cuda")
        P = _device.ptr

        def k_index():  # K3: the index a deserialized stream's decode computes
            rc = L.szx_index_f32(P(p["constant_map"]), P(p["mu"]), P(s._req), P(s._codes), n,
                                 bs, P(idx3), P(st4), P(st4) + 16, P(isc), isc.numel(), sp)
            assert rc == 0

        def k_decode():
            rc = L.szx_decompress_indexed_f32(P(p["constant_map"]), P(p["mu"]), P(s._req),
                                              P(s._codes), P(s._mid_buf), s.mid_len, n, bs,
                                              P(idx3), P(out), P(st4) + 24, sp)
            assert rc == 0

        def timed(fn):
            evs = []
            for _ in range(args.kernel_reps):
                flush.zero_()
                a0 = torch.cuda.Event(enable_timing=True)
                a1 = torch.cuda.Event(enable_timing=True)
                a0.record(stream)
                fn()
                a1.record(stream)
                evs.append((a0, a1))
            torch.cuda.synchronize()
            return statistics.median(a0.elapsed_time(a1) for a0, a1 in evs)

        k_index()
        k_decode()
        kt["index128_kernel"] = timed(k_index)
        kt["decode128_kernel"] = timed(k_decode)
        kt["compress128_kernel"] = timed(lambda: compress_device(x, n, bs, head["e"], pools,
                                                                 small, sp, s._index))
        if dist is not None:
            tk = torch.tensor([kt[k] for k in sorted(kt)], dtype=torch.float64, device="cuda")
            dist.all_reduce(tk, op=dist.ReduceOp.MAX)
            kt = dict(zip(sorted(kt), (float(v) for v in tk.cpu())))
        del idx3, isc
    tc_ms, td_ms, c_bytes = head["tc_ms"], head["td_ms"], head["c"]
    comp_traffic, dec_traffic = N4 + c_bytes, c_bytes + N4
    comp_gbs_alg = comp_traffic / (tc_ms * 1e-3) / 1e9
    dec_gbs_alg = dec_traffic / (td_ms * 1e-3) / 1e9
    value = ws * 2 * N4 / ((tc_ms + td_ms) * 1e-3) / 1e9

    # ---- e2e through the C-ABI host-buffer entry points (pinned host memory) -----------
    e2e = None
    if args.e2e_steps > 0:
        xh = torch.empty(n, dtype=torch.float32, pin_memory=True)
        xh.copy_(x)
        cap = int(L.szx_compress_bound(n, len(dims), bs))
        blob = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
        outh = torch.empty(n, dtype=torch.float32, pin_memory=True)
        dims_c = (ctypes.c_uint64 * len(dims))(*dims)
        olen = ctypes.c_uint64()

        def e2e_compress():
            rc = L.szx_compress_host(xh.data_ptr(), dims_c, len(dims), bs, 1, args.rel,
                                     blob.data_ptr(), cap, ctypes.byref(olen))
            assert rc == 0, _abi.last_error()

        def e2e_decompress():
            rc = L.szx_decompress_host(blob.data_ptr(), olen.value, outh.data_ptr(), n)
            assert rc == 0, _abi.last_error()

        for _ in range(2):
            e2e_compress()
            e2e_decompress()
        if dist is not None:
            dist.barrier()
        tce, tde = [], []
        for _ in range(args.e2e_steps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            e2e_compress()
            t1 = time.perf_counter()
            e2e_decompress()
            t2 = time.perf_counter()
            tce.append(t1 - t0)
            tde.append(t2 - t1)
        te = torch.tensor([sum(tce), sum(tde)], dtype=torch.float64, device="cuda")
        if dist is not None:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        tce_s, tde_s = (float(v) / args.e2e_steps for v in te.cpu())
        blob_len = int(olen.value)
        # the e2e stream must equal the device path's bytes for the same field
        if ws == 1:
            dev_blob = szx.serialize(head["stream"])
            assert dev_blob == blob[:blob_len].numpy().tobytes()
        e2e = {"value": round(ws * 2 * N4 / (tce_s + tde_s) / 1e9, 3), "unit": UNIT,
               "h2d_bytes_per_step": N4 + blob_len, "d2h_bytes_per_step": blob_len + N4,
               "compress_gbs": round(N4 / tce_s / 1e9, 3),
               "decompress_gbs": round(N4 / tde_s / 1e9, 3),
               "ms_per_step": round(1e3 * (tce_s + tde_s), 3),
               "path": "szx_compress_host + szx_decompress_host (pinned host buffers)"}

    # ---- CPU baseline (rank 0, N=1 only) -------------------------------------------------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        ns = min(args.cpu_sample, n)
        cpu = cpu_baseline(x[:ns].cpu().numpy(), head["e"])

    # ---- traffic from a committed ncu capture of this workload, if present --------------
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        traffic = t.get(args.config, {})
    except Exception:
        traffic = {}

    # ---- roofline of the dominant kernel: algorithmic bytes per launch / its device time --
    C = c_bytes
    nb_h = -(-n // bs)
    idx_bytes = (-(-nb_h // 8) + 4 * nb_h + head["n_nc"] + -(-2 * head["m"] // 8) +
                 64 * (-(-nb_h // 64) + 1))
    alg = {"compress128_kernel": N4 + C, "decode128_kernel": C + N4, "index128_kernel": idx_bytes}
    if not kt:
        kt = {"compress128_kernel": tc_ms, "decode128_kernel": td_ms}
    per_kernel = {k: {"ms": round(v, 4), "bytes": alg[k],
                      "gbs": round(alg[k] / (v * 1e-3) / 1e9, 2),
                      "frac": round(alg[k] / (v * 1e-3) / 1e9 / hbm_peak, 4)}
                  for k, v in kt.items()}
    dom = max(kt, key=lambda k: kt[k])
    for k in per_kernel:
        per_kernel[k]["traffic"] = traffic.get(k)
    roof = {"bound": "hbm", "kernel": dom, "achieved": per_kernel[dom]["gbs"], "peak": hbm_peak,
            "unit": "GB/s", "frac": per_kernel[dom]["frac"], "traffic": traffic.get(dom),
            "peak_source": peak_src, "algorithmic_bytes": alg[dom],
            "algorithmic_bytes_rule": "compress: 4N read + C write; decode: C read + 4N write; "
                                      "index: map+mu+req+codes read + index entries written",
            "per_kernel": per_kernel,
            "step_ms": {"compress": round(tc_ms, 4), "decompress": round(td_ms, 4),
                        "decompress_from_bytes_k3_plus_k2": (
                            round(kt["index128_kernel"] + kt["decode128_kernel"], 4)
                            if "index128_kernel" in kt else None)}}

    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(tc_ms + td_ms, 4), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg["name"], "dims": list(dims), "n_values_per_gpu": n,
                   "rel_eb": args.rel, "block_size": bs,
                   "parallelism": f"shard{ws}" if ws > 1 else "single",
                   "l2": (f"input {N4 / 2**20:.0f} MiB "
                          f"{'>' if N4 > L2_BYTES else '<'} L2; 252 MiB L2 flush before each "
                          "timed kernel"),
                   "step": "compress (K1, which also writes the decode index) + decompress (K2 "
                           "through that index), device events; a deserialized stream's "
                           "decompress adds K3 (index128_kernel, step_ms.decompress_from_bytes)"},
        "compress_gbs": round(ws * N4 / (tc_ms * 1e-3) / 1e9, 3),
        "decompress_gbs": round(ws * N4 / (td_ms * 1e-3) / 1e9, 3),
        "cr": round(N4 / c_bytes, 4),
        "compressed_bytes": c_bytes,
        "max_abs_err_over_eb": round(head["err"] / head["e"], 6),
        "roofline": roof,
        "sweep": {str(r): {"compress_gbs": round(ws * N4 / (v["tc_ms"] * 1e-3) / 1e9, 3),
                           "decompress_gbs": round(ws * N4 / (v["td_ms"] * 1e-3) / 1e9, 3),
                           "cr": round(N4 / v["c"], 4),
                           "max_abs_err_over_eb": round(v["err"] / v["e"], 6),
                           "parity": v["parity"]}
                  for r, v in results.items()},
        "e2e": e2e,
        "cpu_baseline": cpu,
        # our kernels inside timed regions: K1 per compress, K2 per decompress, the per-kernel
        # timing reps (K3, K2, K1), and per e2e round trip what the host entries launch
        # (host_launches: K0 + K1 chunks; K3 over the first chunk, K3, the plan, K2 per chunk)
        "gpu_launches": 2 * args.steps * len(results) + 3 * args.kernel_reps +
                        (host_launches(L, n, bs) * args.e2e_steps if e2e else 0),
        "clocks": head["clocks"],
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
