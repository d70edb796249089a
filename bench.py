#!/usr/bin/env python3
"""Benchmark of the AHS hot path on B200: features -> select -> sort.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg5_r32] [--impl ours|reference]

One step = one pass of the whole hot path (ahs_features, ahs_select, ahs_sort)
over the workload's keys, resident in HBM.  The default workload is the
largest BASELINE.json config (cfg5 r=32: 2^28 (uint32 key, uint32 value)
pairs, keys uniform over 32 bits, GENERAL branch, 2 GiB), above BASELINE's
n >= 2^26 gate; a second headline block (`headline_keys`) times the
keys-only GENERAL config cfg4a (2^26 int32).  L2 is flushed (256 MiB write)
before every timed step.  Timing: CUDA
events on the launching stream around each step, barrier + synchronize around
the timed region, max over ranks.  N > 1 runs independent replicas (one per
GPU, weak scaling; the method has no cross-GPU exchange: DESIGN.md §7).

Prints ONE JSON line on rank 0.  `--impl reference` times the CPU oracle
(the only reference this paper has: PAPER.md has no code) on a bounded
sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

METRIC = "sorted keys/sec (Gkeys/s) per strategy on 1 B200; achieved HBM GB/s vs roofline"
L2_FLUSH_BYTES = 256 << 20


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
              "utilization.gpu")

    def __init__(self, gpu: int):
        self.gpu, self.proc, self.lines = gpu, None, []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, smax, reasons, loaded = [], None, set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                c, cm, util = float(parts[0]), float(parts[1]), float(parts[8])
            except ValueError:
                continue
            smax = cm
            sm.append(c)
            if util > 0:
                loaded.append(c)
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        use = loaded or sm
        out = {"sm_mhz": statistics.median(use) if use else None, "sm_max_mhz": smax,
               "reasons": sorted(reasons), "samples": len(sm), "samples_under_load": len(loaded),
               "window": "soak + timed steps"}
        if not sm:
            out["raw"] = self.lines[:3]
        return out


# ------------------------------------------------------------ distributed
def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if ws > 1:
        import torch.distributed as dist
        backend = "gloo" if args.cpu_dist else "nccl"
        dist.init_process_group(backend)
        pg = dist
    return ws, rank, local, pg


def dist_max(pg, x: float, device) -> float:
    if pg is None:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


def barrier(pg):
    if pg is not None:
        pg.barrier()


# --------------------------------------------------------- oracle (CPU)
def host_info():
    """CPU model, logical CPU count and the affinity the process started with."""
    model = None
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        aff = sorted(os.sched_getaffinity(0))
    except (AttributeError, OSError):
        aff = None
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "affinity_cpus": len(aff) if aff else None}


def cpu_oracle_rate(keys, vals, budget_s: float, max_n: int):
    """Time the oracle pipeline (features -> FSM -> sort) on a bounded prefix, pinned to one
    core (sched_setaffinity) for the duration: the oracle is single-threaded C."""
    import oracle
    n = min(keys.size, max_n)
    k, v = keys[:n].copy(), (vals[:n].copy() if vals is not None else None)
    pinned = None
    try:
        old = os.sched_getaffinity(0)
        pinned = min(old)
        os.sched_setaffinity(0, {pinned})
    except (AttributeError, OSError):
        old = None
    times = []
    try:
        t_end = time.perf_counter() + budget_s
        while True:
            t0 = time.perf_counter()
            oracle.ahs(k, v)
            times.append(time.perf_counter() - t0)
            if time.perf_counter() > t_end or len(times) >= 10:
                break
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)
    med = statistics.median(times)
    return n / med / 1e9, n, len(times), med, pinned


# ------------------------------------------------------------ GPU timing
def upload(torch, a: np.ndarray, device):
    if a.dtype in (np.int64, np.uint64):  # NEXT-3 64-bit keys
        t = torch.from_numpy(a.view(np.int64)).to(device)
        return t.view(torch.uint64) if a.dtype == np.uint64 else t
    t = torch.from_numpy(a.view(np.int32)).to(device)
    return t.view(torch.uint32) if a.dtype == np.uint32 else t


def time_pipeline(torch, ahs, keys_np, vals_np, steps, warmup, device, flush, profile=False,
                  pg=None, soak_s=0.0, sampler=None):
    n = keys_np.size
    dk = upload(torch, keys_np, device)
    dv = upload(torch, vals_np, device) if vals_np is not None else None
    ko = torch.empty_like(dk)
    vo = torch.empty_like(dv) if dv is not None else None
    ws = ahs.Workspace(n, dv is not None, device, key_dtype=keys_np.dtype)
    stream = torch.cuda.current_stream(device)

    def step():
        f = ahs.ahs_features(dk, ws, stream)
        s, r = ahs.ahs_select(f)
        ahs.ahs_sort(dk, dv, ko, vo, s, f, ws, stream)
        return f, s, r

    for _ in range(warmup):
        flush.zero_()
        f, s, r = step()
    torch.cuda.synchronize(device)
    if sampler:
        sampler.start()
        time.sleep(0.5)  # nvidia-smi start-up
    if soak_s > 0:  # untimed load so the clock sampler sees the GPU under this workload
        t_end = time.perf_counter() + soak_s
        while time.perf_counter() < t_end:
            flush.zero_()
            step()
        torch.cuda.synchronize(device)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    barrier(pg)
    torch.cuda.synchronize(device)
    launches0 = ahs.ahs_launch_count()
    for i in range(steps):
        flush.zero_()
        ev[i][0].record(stream)
        f, s, r = step()
        ev[i][1].record(stream)
    torch.cuda.synchronize(device)
    launches = ahs.ahs_launch_count() - launches0
    barrier(pg)
    total_ms = sum(a.elapsed_time(b) for a, b in ev)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    prof = None
    if profile:
        # per-kernel durations: a second timed pass of the same steps with CUDA
        # events around every launch (they add launch overhead, so the headline
        # step time above is taken without them)
        ahs.ahs_profile_begin()
        for i in range(steps):
            flush.zero_()
            step()
        torch.cuda.synchronize(device)
        ahs.ahs_profile_end()
        prof = ahs.ahs_profile_read()
    clocks = sampler.stop() if sampler else None
    passes = ahs.ahs_sort_passes(f, s, dv is not None)
    executed = ahs.ahs_sort_executed_passes(ws, stream) if passes > 0 else 0
    digit_passes, bucket_local = ahs.ahs_sort_plan(ws, stream) if passes > 0 else (0, 0)
    if executed < 0:  # no device plan on this path (COUNTING): the nominal passes all run
        executed = digit_passes = passes
    return dict(total_ms=total_ms, f=f, s=s, r=r, launches=launches, prof=prof, passes=passes,
                executed=executed, digit_passes=digit_passes, bucket_local=bucket_local, clocks=clocks,
                step_ms=step_ms)


def entropy_exact_report(torch, ahs, keys_np, vals_np, device, reps=5):
    """NEXT-2: the paper-literal entropy (over distinct values) of the sorted output, the FSM
    branch it would give under the paper's own normalisation (RANGE: 0.7 log2 k), and the
    K8 kernel's time (it reads the 4n-byte output about twice)."""
    n = keys_np.size
    dk = upload(torch, keys_np, device)
    ws = ahs.Workspace(n, False, device)
    stream = torch.cuda.current_stream(device)
    f = ahs.ahs_features(dk, ws, stream)
    s, r = ahs.ahs_select(f)
    ko = torch.empty_like(dk)
    ahs.ahs_sort(dk, None, ko, None, s, f, ws, stream)
    hx = ahs.ahs_entropy_sorted(ko, ws, stream)
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        ahs.ahs_entropy_sorted(ko, ws, stream)  # synchronizes
        b.record(stream)
        torch.cuda.synchronize(device)
        ts.append(a.elapsed_time(b))
    ms = statistics.median(ts)
    fp = ahs.Features.from_buffer_copy(f)
    fp.entropy = hx
    sp, rp = ahs.ahs_select(fp, ahs.ahs_thresholds_default(entropy_norm=1))
    return {"H_exact": hx, "H16": f.entropy, "branch": ahs.STRATEGY_NAMES[s],
            "branch_paper_literal": ahs.STRATEGY_NAMES[sp], "agree": sp == s,
            "ms": ms, "GBps_one_read": 4 * n / (ms * 1e-3) / 1e9,
            "note": "K8 ahs_entropy_sorted on ahs_sort's output, incl. its 8-byte readback; "
                    "paper-literal FSM = RANGE norm (0.7 log2 k) with H over distinct values"}


def segments_report(torch, ahs, device, reps=10):
    """NEXT-4: ahs_sort_segments on two segment-length mixes (L2 flushed per run): the
    paper's small-n regime (2^20 segments of 1..20 keys: Listing 1's insertion sort, one
    thread per segment) and 2^13 segments of 1000..2048 keys (one CTA each).  Algorithmic
    bytes: read + write of keys (and values) + the offsets."""
    rows = []
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=device)
    for name, nseg, lo, hi, kv in (("insertion_1_20", 1 << 20, 1, 20, False),
                                   ("insertion_1_20_kv", 1 << 20, 1, 20, True),
                                   ("radix_1000_2048", 1 << 13, 1000, 2048, False)):
        lens = np.random.default_rng(7).integers(lo, hi + 1, nseg)
        off = np.zeros(nseg + 1, dtype=np.int64)
        off[1:] = np.cumsum(lens)
        n = int(off[-1])
        keys = (synth.stream(5, n) >> np.uint64(32)).astype(np.uint32).view(np.int32)
        dk = upload(torch, keys, device)
        dv = torch.arange(n, dtype=torch.int32, device=device).view(torch.uint32) if kv else None
        ko, vo = torch.empty_like(dk), (torch.empty_like(dv) if kv else None)
        doff = torch.from_numpy(off.astype(np.uint32).view(np.int32)).to(device)
        bad = torch.zeros(1, dtype=torch.int32, device=device)
        for _ in range(3):
            ahs.ahs_sort_segments(dk, dv, ko, vo, doff, hi, bad)
        torch.cuda.synchronize(device)
        ts = []
        for _ in range(reps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ahs.ahs_sort_segments(dk, dv, ko, vo, doff, hi, bad)
            b.record()
            torch.cuda.synchronize(device)
            ts.append(a.elapsed_time(b))
        ms = statistics.median(ts)
        byts = n * (8 + (8 if kv else 0)) + 4 * (nseg + 1)
        rows.append({"case": name, "segments": nseg, "n": n, "kv": kv, "max_segment": hi, "us": ms * 1e3,
                     "Gkeys_s": n / (ms * 1e-3) / 1e9, "GBps": byts / (ms * 1e-3) / 1e9,
                     "bad": int(bad.item())})
    return rows


def time_e2e(torch, ahs, keys_np, vals_np, steps, warmup, device):
    """Same metric through the C-ABI host entry point: pinned host buffers, every step's H2D
    and D2H inside the timed region.  Steps rotate over three streams, each with its own
    device scratch, pinned output buffers and host thread, through ahs_sort_host_async: one
    step's D2H overlaps the next steps' H2D and compute (PCIe is full duplex), and a thread
    waiting in its step's features round trip does not hold back the others' uploads; a
    stream is synchronized before its buffers are reused, three steps later, so the upload
    engine never waits for a download.  Device time: events on every stream, from a start
    event all wait on to the latest end event."""
    n = keys_np.size
    w = np.int64 if keys_np.itemsize == 8 else np.int32
    hk = torch.from_numpy(keys_np.view(w)).pin_memory()
    hv = torch.from_numpy(vals_np.view(np.int32)).pin_memory() if vals_np is not None else None
    NB = 3  # streams / buffers / host threads in flight (4 or 6: no faster, r01_summary.md)
    hko = [torch.empty_like(hk).pin_memory() for _ in range(NB)]
    hvo = [torch.empty_like(hv).pin_memory() if hv is not None else None for _ in range(NB)]
    udt = {np.dtype(np.uint32): torch.uint32, np.dtype(np.uint64): torch.uint64}.get(keys_np.dtype)
    if udt is not None:
        hk, hko = hk.view(udt), [t.view(udt) for t in hko]
    if hv is not None:
        hv, hvo = hv.view(torch.uint32), [t.view(torch.uint32) for t in hvo]
    nb = ahs.ahs_host_scratch_bytes(n, hv is not None, keys_np.dtype)
    scratch = [torch.empty(nb, dtype=torch.uint8, device=device) for _ in range(NB)]
    streams = [torch.cuda.Stream(device) for _ in range(NB)]
    start = torch.cuda.Event(enable_timing=True)
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(NB)]
    errors = []
    ready, go = threading.Barrier(NB + 1), threading.Barrier(NB + 1)

    def worker(b):  # one host thread per stream: it blocks in its step's features round trip
        try:  # while the other threads' steps keep the copy engines busy
            torch.cuda.set_device(device)
            for _ in range(max(1, warmup // NB)):  # per-thread warm-up (the library's per-thread
                ahs.ahs_sort_host(hk, hv, hko[b], hvo[b], scratch[b], stream=streams[b])  # host buffer)
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)
        ready.wait()
        go.wait()
        try:
            for i in range(b, steps, NB):
                if i >= NB:
                    streams[b].synchronize()  # step i - NB used these buffers
                ahs.ahs_sort_host(hk, hv, hko[b], hvo[b], scratch[b], stream=streams[b], sync=False)
            ends[b].record(streams[b])
        except Exception as e:  # pragma: no cover - reported below
            errors.append(e)

    threads = [threading.Thread(target=worker, args=(b,)) for b in range(NB)]
    for t in threads:
        t.start()
    ready.wait()
    torch.cuda.synchronize(device)
    start.record(streams[0])
    for b in range(1, NB):
        streams[b].wait_event(start)
    go.wait()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    torch.cuda.synchronize(device)
    ms = max(start.elapsed_time(e) for e in ends)
    last = hko[(steps - 1) % NB].view(torch.int64 if keys_np.itemsize == 8 else torch.int32).numpy().view(keys_np.dtype)
    if not bool((last[1:] >= last[:-1]).all()):  # the host output of the last step is sorted
        raise RuntimeError("e2e: ahs_sort_host_async produced unsorted output")
    kb = keys_np.itemsize
    nbi = n * kb + (n * 4 if hv is not None else 0)
    return ms, nbi, nbi


def sort_bytes(strategy: int, passes: int, n: int, kv: bool, shift: int = 1, kb: int = 4) -> int:
    """Algorithmic HBM bytes of ahs_sort: per executed pass read + write of
    the keys (2 kb n, kb = key bytes) and values (8n); counting keys-only = write kb n.
    K5 reads no keys for 32-bit keys; for 64-bit keys K5b reads them once (8n) when the
    feature buckets are coarser than 16 bits (shift > 16)."""
    if passes == 0:
        return kb * n if strategy == 0 else 0
    hist = kb * n if (kb == 8 and shift > 16) else 0
    return hist + passes * (2 * kb + (8 if kv else 0)) * n


def contract_bytes(strategy: int, passes_nominal: int, n: int, kv: bool, kb: int = 4) -> int:
    """BASELINE.json's contract roofline bytes: radix / GENERAL (2p + 1) bytes n with
    the nominal pass count p and bytes = key bytes (+ 4 per value: BJ counts 8 for 32-bit pairs, which
    over-counts the histogram read by 4n); counting: a read and a write of the keys (and values)."""
    bytes_per = kb + (4 if kv else 0)
    if strategy == 0 and passes_nominal <= 1:
        return 2 * bytes_per * n
    return (2 * passes_nominal + 1) * bytes_per * n


def traffic_from_profiles(workload: str):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, from the
    committed `ncu --set full` capture of that workload (profiles/ncu_traffic.json)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(p))
        return d.get(workload, {}).get("onesweep_dram_bytes_per_launch")
    except Exception:
        return None


PER_LAUNCH_BYTES = {"onesweep": 8, "onesweep_kv": 16, "count_fill": 4, "count_scatter_kv": 16,
                    "radix_hist": 4, "feat_reduce": 4, "feat_hist": 4}


def dominant_roofline(res, n, kv, kb, workload, peak, peak_kind):
    """Roofline of the step's dominant kernel (the onesweep digit pass): algorithmic bytes per
    launch (read + write of every key and value) / its mean CUDA-event launch time."""
    prof = res["prof"]
    kname = "onesweep_kv" if kv else "onesweep"
    if prof.get(kname, {}).get("launches", 0) == 0:
        kname = max(prof, key=lambda k: prof[k]["ms"])
    kl = prof[kname]["launches"]
    if kname.startswith("onesweep") and res["digit_passes"] < res["passes"]:
        # launches the plan skips return at once (NEXT-1; the bucket-local plan's unused passes)
        kl = kl * res["digit_passes"] // res["passes"]
    kms = prof[kname]["ms"] / max(1, kl)
    per = PER_LAUNCH_BYTES.get(kname, 4) * n
    if kname.startswith("onesweep") and kb == 8:
        per = (16 + (8 if kv else 0)) * n
    achieved = per / (kms * 1e-3) / 1e9
    return {"bound": "hbm", "kernel": kname, "achieved": round(achieved, 1), "peak": peak,
            "peak_kind": peak_kind, "unit": "GB/s", "frac": round(achieved / peak, 4),
            "traffic": traffic_from_profiles(workload), "algorithmic_bytes_per_launch": per,
            "ms_per_launch": kms,
            "timing": "CUDA events around every launch on the launching stream, second timed pass of the "
                      "same K steps (the headline value is timed without them)"}


def table_row(torch, ahs, cfg, k2, v2, steps, device, flush, peak, skip=True, count_single=False):
    """One per-strategy row: pipeline and sort throughput, fractions of the roofline.  With
    skip=False the NEXT-1 trivial-pass skipping is off: every nominal pass executes (the
    contract row of SURVEY §8(d)); with skip=True the row is the NEXT-1 row."""
    prev = ahs.ahs_set_skip_trivial(-1)
    prev_cs = ahs.ahs_set_count_kv_single(-1)
    prev_bl = ahs.ahs_set_bucket_local(-1)
    ahs.ahs_set_skip_trivial(1 if skip else 0)
    ahs.ahs_set_count_kv_single(1 if count_single else 0)
    ahs.ahs_set_bucket_local(1 if skip else 0)  # the contract row (skip off) runs the classic plan
    try:
        r2 = time_pipeline(torch, ahs, k2, v2, steps, 2, device, flush, profile=True)
    finally:
        ahs.ahs_set_skip_trivial(prev)
        ahs.ahs_set_count_kv_single(prev_cs)
        ahs.ahs_set_bucket_local(prev_bl)
    p2 = r2["prof"]
    n2 = k2.size
    kv2 = v2 is not None
    sort_ms2 = sum(v["ms"] for k, v in p2.items() if not k.startswith("feat")) / steps
    feat_ms2 = sum(v["ms"] for k, v in p2.items() if k.startswith("feat")) / steps
    kb2 = k2.dtype.itemsize
    sb2 = sort_bytes(r2["s"], r2["executed"], n2, kv2, r2["f"].shift, kb2)
    row = {
        "workload": cfg, "n": n2, "kv": kv2, "strategy": ahs.STRATEGY_NAMES[r2["s"]],
        "rule": ahs.RULE_NAMES[r2["r"]], "skip_trivial": skip, "passes": r2["passes"],
        "count_kv_single": count_single, "bucket_local": bool(r2["bucket_local"]),
        "digit_passes_executed": r2["digit_passes"],
        "passes_executed": r2["executed"],
        "pipeline_Gkeys_s": n2 * steps / (r2["total_ms"] * 1e-3) / 1e9,
        "sort_Gkeys_s": n2 / (sort_ms2 * 1e-3) / 1e9 if sort_ms2 > 0 else None,
        "sort_GBps": sb2 / (sort_ms2 * 1e-3) / 1e9 if sort_ms2 > 0 else None,
        "sort_frac_of_peak": (sb2 / (sort_ms2 * 1e-3) / 1e9) / peak if sort_ms2 > 0 else None,
        "key_bytes": kb2,
        "features_GBps": 2 * kb2 * n2 / (feat_ms2 * 1e-3) / 1e9 if feat_ms2 > 0 else None,
        "kernels_ms": {k: v["ms"] / v["launches"] for k, v in p2.items() if v["launches"]},
    }
    # BASELINE's contract roofline ((2p + 1) bytes n, p nominal) is only meaningful when the
    # nominal passes all ran: skip-on rows that skipped a pass report it as null
    contract_ok = sort_ms2 > 0 and r2["executed"] == r2["passes"]
    cb = contract_bytes(r2["s"], r2["passes"], n2, kv2, kb2)
    row["contract_frac_of_8TBps"] = cb / (sort_ms2 * 1e-3) / 8e12 if contract_ok else None
    row["contract_frac_of_peak"] = cb / (sort_ms2 * 1e-3) / 1e9 / peak if contract_ok else None
    return row, r2


def run_ours(args):
    import torch
    ws, rank, local, pg = dist_setup(args)
    device = torch.device("cuda", local)
    torch.cuda.set_device(device)
    import paper_2506_20677_b200 as ahs
    ahs.lib()
    peak, peak_kind = load_peaks()
    keys, vals, dt = synth.make(args.workload)
    n = keys.size
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=device)
    sampler = ClockSampler(local)
    res = time_pipeline(torch, ahs, keys, vals, args.steps, args.warmup, device, flush, profile=True,
                        pg=pg, soak_s=args.soak, sampler=sampler)
    tmax = dist_max(pg, res["total_ms"], device)
    value = ws * n * args.steps / (tmax * 1e-3) / 1e9
    f, s, r, prof = res["f"], res["s"], res["r"], res["prof"]
    kv = vals is not None
    kb = keys.dtype.itemsize
    roof = dominant_roofline(res, n, kv, kb, args.workload, peak, peak_kind)
    step_total = sum(v["ms"] for v in prof.values())
    # per-kernel numbers come from the profiled pass (steps with per-launch events)
    kernels = {k: {"ms_per_launch": v["ms"] / v["launches"], "launches": v["launches"],
                   "share_of_kernel_time": v["ms"] / step_total}
               for k, v in prof.items() if v["launches"]}
    sb = sort_bytes(s, res["executed"], n, kv, f.shift, kb)
    sort_ms = sum(v["ms"] for k, v in prof.items() if not k.startswith("feat")) / args.steps
    feat_ms = sum(v["ms"] for k, v in prof.items() if k.startswith("feat")) / args.steps

    out = {
        "metric": METRIC, "value": round(value, 4), "unit": "Gkeys/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": tmax / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": dt,
        "data": "synthetic (SplitMix64 recipe of SURVEY.md §8(d))",
        "config": {"workload": args.workload, "n": n, "key_dtype": dt, "kv": kv,
                   "strategy": ahs.STRATEGY_NAMES[s], "rule": ahs.RULE_NAMES[r], "passes": res["passes"],
                   "passes_executed": res["executed"], "digit_passes_executed": res["digit_passes"],
                   "bucket_local": bool(res["bucket_local"]),
                   "l2": "flushed before every timed step (256 MiB write); the inputs are also larger than L2",
                   "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU"},
        "roofline": roof,
        "stages": {"features_ms": feat_ms, "sort_kernels_ms": sort_ms,
                   "sort_algorithmic_bytes": sb,
                   "sort_GBps": sb / (sort_ms * 1e-3) / 1e9 if sort_ms > 0 else None,
                   "sort_frac_of_peak": (sb / (sort_ms * 1e-3) / 1e9) / peak if sort_ms > 0 else None,
                   "step_ms_median": statistics.median(res["step_ms"])},
        "kernels": kernels,
        "gpu_launches": res["launches"],
        "clocks": res["clocks"],
        "features": {"k": f.k, "nbins": f.nbins, "H": f.entropy, "descents": f.descents},
    }
    # second headline: keys-only GENERAL at 2^26 (cfg4a), same protocol, its own roofline
    if args.keys_workload and args.keys_workload != args.workload:
        k4, v4, dt4 = synth.make(args.keys_workload)
        r4 = time_pipeline(torch, ahs, k4, v4, args.steps, args.warmup, device, flush, profile=True, pg=pg)
        t4 = dist_max(pg, r4["total_ms"], device)
        out["headline_keys"] = {
            "workload": args.keys_workload, "n": k4.size, "dtype": dt4, "kv": v4 is not None,
            "strategy": ahs.STRATEGY_NAMES[r4["s"]], "passes_executed": r4["executed"],
            "value": round(ws * k4.size * args.steps / (t4 * 1e-3) / 1e9, 4), "unit": "Gkeys/s",
            "ms_per_step": t4 / args.steps, "gpu_launches": r4["launches"],
            "roofline": dominant_roofline(r4, k4.size, v4 is not None, k4.dtype.itemsize, args.keys_workload,
                                          peak, peak_kind)}
        del k4, v4
    # NEXT-2: paper-literal entropy of the output and the branch it implies
    if rank == 0 and kb == 4:
        out["entropy_exact"] = entropy_exact_report(torch, ahs, keys, vals, device)
    # NEXT-4: batched small-n segment sorts
    if rank == 0 and args.configs:
        out["segments"] = segments_report(torch, ahs, device)
        for r in out["segments"]:
            r["frac_of_peak"] = r["GBps"] / peak
    # end to end through the C ABI with host buffers
    if not args.no_e2e:
        e_steps = max(3, args.steps)  # the same K steps as the device-timed region
        e_ms, bi, bo = time_e2e(torch, ahs, keys, vals, e_steps, 2, device)
        e_max = dist_max(pg, e_ms, device)
        out["e2e"] = {"value": round(ws * n * e_steps / (e_max * 1e-3) / 1e9, 4), "unit": "Gkeys/s",
                      "h2d_bytes_per_step": bi, "d2h_bytes_per_step": bo,
                      "ms_per_step": e_max / e_steps, "api": "ahs_sort_host (pinned host buffers)"}
    # per-strategy table (BASELINE.json metric is per strategy).  Every radix row whose NEXT-1
    # plan skips passes gets a second, contract row with skipping off.
    if args.configs and ws == 1:
        rows = []
        for cfg in [c for c in args.configs.split(",") if c]:
            k2, v2, dt2 = synth.make(cfg)
            row, r2 = table_row(torch, ahs, cfg, k2, v2, args.table_steps, device, flush, peak, skip=True)
            if k2.dtype.itemsize == 4:  # K8 (NEXT-2) is built for 32-bit keys
                ee = entropy_exact_report(torch, ahs, k2, v2, device, reps=2)
                row.update({"H16": ee["H16"], "H_exact": ee["H_exact"],
                            "branch_paper_literal": ee["branch_paper_literal"], "branch_agree": ee["agree"]})
            else:
                row.update({"H16": r2["f"].entropy})
            rows.append(row)
            if r2["executed"] < r2["passes"] or r2["bucket_local"]:
                row_c, _ = table_row(torch, ahs, cfg, k2, v2, args.table_steps, device, flush, peak, skip=False)
                rows.append(row_c)
            if v2 is not None and r2["s"] == 0 and 8 < r2["f"].bits <= 10:
                # key-value COUNTING with 256 < k <= 1024: the opt-in single 10-bit scatter beside the default
                row_s, _ = table_row(torch, ahs, cfg, k2, v2, args.table_steps, device, flush, peak,
                                     count_single=True)
                rows.append(row_s)
            del k2, v2
        out["strategies"] = rows
    # CPU oracle baseline (rank 0, N = 1 only)
    if rank == 0 and ws == 1 and not args.no_cpu:
        rate, ns, reps, med, core = cpu_oracle_rate(keys, vals, args.cpu_budget, args.cpu_sample)
        out["cpu_baseline"] = {"value": round(rate, 6), "unit": "Gkeys/s", "cores": 1, "kind": "oracle",
                               "sample": f"first {ns} keys of {args.workload} ({'pairs' if kv else 'keys'}), "
                                         f"oracle features+FSM+sort, median of {reps} runs ({med:.2f} s each), "
                                         f"one thread pinned to CPU {core}",
                               "host": host_info()}
    if rank == 0:
        print(json.dumps(out))
    if pg is not None:
        pg.destroy_process_group()


def run_reference(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import oracle
    oracle.build()
    keys, vals, dt = synth.make(args.workload)
    ns = min(keys.size, args.ref_sample)
    k, v = keys[:ns].copy(), (vals[:ns].copy() if vals is not None else None)
    for _ in range(args.warmup):
        oracle.ahs(k, v)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.ahs(k, v)
    dt_s = time.perf_counter() - t0
    value = ns * args.steps / dt_s / 1e9
    sample = (f"first {ns} keys of {args.workload} per step (oracle features+FSM+sort, one thread)")
    out = {"impl": "reference", "metric": METRIC, "value": round(value, 6), "unit": "Gkeys/s",
           "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": dt_s * 1e3 / args.steps, "higher_is_better": True, "scaling": "weak",
           "vs_baseline": None, "dtype": dt, "data": "synthetic",
           "config": {"workload": args.workload, "n": keys.size, "sample_n": ns, "key_dtype": dt,
                      "kv": vals is not None},
           "cpu_baseline": {"value": round(value, 6), "unit": "Gkeys/s", "cores": 1, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": round(value, 6), "unit": "Gkeys/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg5_r32", choices=sorted(synth.CONFIGS))
    ap.add_argument("--keys-workload", default="cfg4a", help="second (keys-only) headline block; '' to skip")
    ap.add_argument("--configs", default="cfg1,cfg2,cfg2kv,cfg3,cfg4a,cfg4b,cfg4c,cfg4d,cfg5_r8,cfg5_r16,cfg5_r20,"
                                         "cfg5_r24,cfg5_r28,cfg5_r32,cfg6,cfg6kv,cfg7kv",
                    help="per-strategy table rows (single GPU only); '' to skip")
    ap.add_argument("--table-steps", type=int, default=5)
    ap.add_argument("--soak", type=float, default=2.0, help="untimed seconds of load before timing")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--cpu-sample", type=int, default=1 << 24, help="oracle baseline: first N keys")
    ap.add_argument("--ref-sample", type=int, default=1 << 22)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-dist", action="store_true", help=argparse.SUPPRESS)
    args = ap.parse_args()
    assert args.warmup >= 1
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
