#!/usr/bin/env python
"""Benchmark of the IPS4o hot path on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config H|C1|C2a|C2b|C3_*|C4] [--impl ours|reference]

One step = one in-place ips4o_sort of the whole synthetic workload (all distribution levels
and the base case), inputs resident in HBM.  The input is larger than L2 and is restored
from a pristine device copy before every step, outside the timed region (an in-place sort
destroys its input); each step is bracketed by CUDA events on the sorting stream.

Multi-GPU: the north star is one GPU; N > 1 runs independent replicas (one process per GPU,
each sorting its own copy), value = total elements / max-over-ranks time ("weak" scaling).

--impl reference times the CPU oracle (oracle/, the paper's sequential IS4o written from the
paper) on a bounded sample of the same workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

METRIC = "Gelem/s sorted in-place on 1 B200 (2^28 u64) and % of HBM-pass roofline"

# name -> (distribution, log2 n, description)
CONFIGS = {
    "H": ("uniform", 28, "H: 2^28 u64 keys i.i.d. uniform over [0,2^64), seed 1 (headline)"),
    "C1": ("uniform", 20, "C1: 2^20 u64 uniform, seed 1 (L2-resident)"),
    "C2a": ("f64_uniform", 28, "C2a: 2^28 f64 uniform [0,1), seed 1"),
    "C2b": ("f64_exponential", 28, "C2b: 2^28 f64 exponential(1), seed 1"),
    "C3_rootdup": ("rootdup", 27, "C3: 2^27 u64 RootDup"),
    "C3_twodup": ("twodup", 27, "C3: 2^27 u64 TwoDup"),
    "C3_eightdup": ("eightdup", 27, "C3: 2^27 u64 EightDup"),
    "C3_almostsorted": ("almostsorted", 27, "C3: 2^27 u64 AlmostSorted"),
    "C3_reversesorted": ("reversesorted", 27, "C3: 2^27 u64 ReverseSorted"),
    "C3_zeros": ("zeros", 27, "C3: 2^27 u64 all-zero"),
    "F3_sorted": ("sorted", 27, "f3: 2^27 u64 already sorted (PAPER.md:444 Sorted)"),
    "F3_ones": ("ones", 27, "f3: 2^27 u64 all equal to 1 (PAPER.md:444 Ones)"),
    "C4": ("pair16", 27, "C4: 2^27 Pair16 (u64 key uniform [0,2^32), payload = index)"),
    "C5": ("rec100", 24, "C5: 2^24 100-byte records (10-byte key)"),
    "F3_pair_f64": ("pair_f64", 27, "f3: 2^27 the paper's Pair (f64 key uniform [0,1) + f64 payload)"),
    "F3_quartet": ("quartet_f64", 26, "f3: 2^26 the paper's Quartet (three f64 keys, lexicographic, + payload)"),
    "C4_kv": ("pair16", 27, "C4 as structure of arrays: 2^27 u64 keys uniform [0,2^32) + u64 values = index, "
                            "ips4o_sort_kv (in place)"),
}
DTYPE = {W.ELEM_U64: "u64", W.ELEM_F64: "f64", W.ELEM_PAIR: "u64x2", W.ELEM_REC100: "u8x100",
         W.ELEM_PAIR_F64: "f64x2", W.ELEM_QUARTET_F64: "f64x4"}
BW_NOMINAL = 8000.0  # GB/s, the north star's "roughly 8 TB/s"


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", d
    return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)", {}


def levels_for(n: int, esize: int) -> int:
    """L = ceil(log_256(n / n_base)), n_base = 4096 (2048 for 100-byte records)."""
    nb = 2048 if esize == 100 else 4096
    if n <= nb:
        return 1
    return max(1, math.ceil(math.log(n / nb, 256) - 1e-12))


# ------------------------------------------------------------------ clocks sampler

class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region: NVML every 4 ms (at
    least ~20 samples in a 0.1 s region), else nvidia-smi every 200 ms."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.out = []
        self.nv = None
        self.mx = 0
        self.stop = threading.Event()
        self.thr = None

    def prepare(self):
        """NVML initialised ahead of the timed region (nvmlInit can take longer than the region)."""
        if self.nv is not None:
            return
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
            nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
            self.nv = (nv, h)
        except Exception:
            self.nv = None

    def __enter__(self):
        self.prepare()
        if self.nv is not None:
            self.thr = threading.Thread(target=self._nvml, daemon=True)
            self.thr.start()
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thr = threading.Thread(target=self._read, daemon=True)
            self.thr.start()
        except Exception:
            self.proc = None
        return self

    def _nvml(self):
        nv, h = self.nv
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        mx = self.mx
        while not self.stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                act = ["Active" if (r & b) else "Not Active" for b in bits]
                self.out.append(",".join([str(sm), str(mx)] + act))
            except Exception:
                pass
            time.sleep(0.004)

    def _read(self):
        for line in self.proc.stdout:
            self.out.append(line.strip())

    def __exit__(self, *a):
        self.stop.set()
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thr:
            self.thr.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        for line in self.out:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(self.NAMES, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            # no sample landed inside the region (NVML missing or failing): one nvidia-smi query now,
            # right behind the region, marked as such
            try:
                line = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                       "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                      timeout=20).stdout.strip().splitlines()[0]
                parts = [p.strip() for p in line.split(",")]
                rs = [nm for nm, v in zip(self.NAMES, parts[2:6]) if v.lower().startswith("active")]
                return {"sm_mhz": float(parts[0]), "sm_max_mhz": float(parts[1]), "reasons": sorted(rs),
                        "samples": 1, "source": "nvidia-smi, one query right after the timed region"}
            except Exception:
                return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml 4 ms" if self.nv else "nvidia-smi 200 ms"}


# ------------------------------------------------------------------ helpers

def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def make_input(cfg: str, n_override: int | None = None):
    dist, e, desc = CONFIGS[cfg]
    n = n_override or (1 << e)
    et, a = W.make(dist, n, 1)
    return et, a, desc


def host_to_device(a: np.ndarray, et: int):
    import torch
    if et in (W.ELEM_F64, W.ELEM_PAIR_F64, W.ELEM_QUARTET_F64):
        return torch.from_numpy(a).cuda()
    if et in (W.ELEM_U64, W.ELEM_PAIR):
        return torch.from_numpy(a.view(np.int64)).cuda().view(torch.uint64)
    return torch.from_numpy(a).cuda()


# ------------------------------------------------------------------ reference arm

def run_reference(args):
    """The oracle as it stands on the host cores, on bounded samples of the workload."""
    import oracle
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    dist, e, desc = CONFIGS[args.config]
    n_full = 1 << e
    sample = min(n_full, 1 << args.ref_log2)
    et, a = W.make(dist, sample, 1)
    esize = W.ELEM_SIZE[et]
    for _ in range(args.warmup):
        oracle.sort(a[: min(sample, 1 << 16)])
    times = []
    for _ in range(args.steps):
        b = a.copy()
        t0 = time.perf_counter()
        oracle.sort_inplace(b)
        times.append(time.perf_counter() - t0)
    t = statistics.mean(times)
    val = sample / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "Gelem/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": DTYPE[et],
        "data": "synthetic",
        "config": {"workload": desc, "n": n_full, "elem_bytes": esize, "sample_n": sample},
        "cpu_baseline": {"value": val, "unit": "Gelem/s", "cores": 1, "kind": "oracle",
                         "sample": f"{dist} n=2^{int(math.log2(sample))} (seed 1) per step, "
                                   f"oracle/ sequential IS4o, 1 thread"},
        "e2e": {"value": val, "unit": "Gelem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(dist: str, log2: int, secs_target: float = 15.0):
    """Oracle on a bounded sample (rank 0, N=1 only)."""
    import oracle
    n = 1 << log2
    et, a = W.make(dist, n, 1)
    b = a.copy()
    t0 = time.perf_counter()
    oracle.sort_inplace(b)
    t = time.perf_counter() - t0
    reps = 1
    # context: the library sort of the same sample on one core (numpy's sort, standing in
    # for std::sort), and the host the numbers come from
    c = a.copy()
    t1 = time.perf_counter()
    if et == W.ELEM_REC100:
        np.sort(np.ascontiguousarray(c).view("S100").ravel())
    elif et == W.ELEM_PAIR:
        np.sort(c.view([("k", "<u8"), ("v", "<u8")]).ravel(), order=["k"])
    elif et in (W.ELEM_PAIR_F64, W.ELEM_QUARTET_F64):
        nk = 1 if et == W.ELEM_PAIR_F64 else 3
        c[np.lexsort(tuple(c[:, j] for j in reversed(range(nk))))]
    else:
        c.sort()
    t_lib = time.perf_counter() - t1
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            model = next((l.split(":", 1)[1].strip() for l in f if l.startswith("model name")), "")
    except OSError:
        pass
    return {"value": n / t / 1e9, "unit": "Gelem/s", "cores": 1, "kind": "oracle",
            "sample": f"{dist} n=2^{log2} (seed 1), {reps} run, {t:.1f} s; oracle/ sequential IS4o "
                      f"(PAPER.md:419), 1 thread",
            "library_sort_1core_gelems": n / t_lib / 1e9, "nproc": os.cpu_count(), "cpu_model": model}


def cpu_parallel_baseline(a: np.ndarray, et: int):
    """The multi-core CPU IPS4o (cpu_baseline/: the paper's parallel
    algorithm with OpenMP threads) on the FULL workload, all host
    cores; median of 3 runs on fresh copies.  Context, not the target."""
    import cpu_baseline
    t = os.cpu_count() or 1
    times = []
    warm = a[: min(a.shape[0], 1 << 16)].copy()
    cpu_baseline.sort_inplace(warm, t)
    for _ in range(3):
        b = a.copy()
        t0 = time.perf_counter()
        cpu_baseline.sort_inplace(b, t)
        times.append(time.perf_counter() - t0)
    ts = statistics.median(times)
    ok = bool(np.all(b[1:] >= b[:-1])) if et in (W.ELEM_U64, W.ELEM_F64) else None
    return {"value": a.shape[0] / ts / 1e9, "unit": "Gelem/s", "cores": t, "kind": "ips4o_cpu",
            "sample": f"the full workload (n={a.shape[0]}), median of 3 runs, {t} OpenMP threads; "
                      "cpu_baseline/ parallel IPS4o (not the oracle)",
            "sorted_check": ok, "ms": ts * 1e3}


# ------------------------------------------------------------------ our arm

def run_ours(args):
    import torch
    import paper_1705_02257_b200 as ips4o

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ips4o.lib()
    et, a, desc = make_input(args.config, args.n)
    n = a.shape[0]
    esize = W.ELEM_SIZE[et]
    kv = args.config.endswith("_kv")
    if kv:
        # structure of arrays: row 0 the keys, row 1 the values (each row contiguous)
        import numpy as _np
        pristine = torch.from_numpy(_np.ascontiguousarray(a.T).view(_np.int64)).cuda().view(torch.uint64)
    else:
        pristine = host_to_device(a, et)
    ver = OracleVerify(a, et) if (rank == 0 and not args.no_verify) else None
    work = pristine.clone()
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream

    def one_sort():
        if kv:
            ips4o.ips4o_sort_kv(work[0].data_ptr(), work[1].data_ptr(), n, W.ELEM_U64, sptr)
        else:
            ips4o.ips4o_sort(work.data_ptr(), n, et, sptr)

    for _ in range(max(args.warmup, 0)):
        work.copy_(pristine)
        one_sort()
    torch.cuda.synchronize()

    # timed region: K steps, per-step events around the sort only (the per-kernel events
    # of the roofline line cost ~1.4 % of a step, so they are recorded in a second K-step
    # region right after this one, same workload and launches)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    clk = ClockSampler(local)
    clk.prepare()
    launches = 0
    stats = None
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    with clk:
        for i in range(args.steps):
            work.copy_(pristine)
            evs[i][0].record(stream)
            one_sort()
            evs[i][1].record(stream)
            stats = ips4o.ips4o_last_stats()
            launches += stats["kernel_launches"]
        torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    step_ms = [s.elapsed_time(e) for s, e in evs]
    # per-kernel durations: the same K steps again with the library's per-launch events
    prof = {}
    if not args.no_kernel_events:
        ips4o.ips4o_profile_enable(True)
        ips4o.ips4o_profile_read()  # clear
        for i in range(args.steps):
            work.copy_(pristine)
            one_sort()
        torch.cuda.synchronize()
        prof = ips4o.ips4o_profile_read()
        ips4o.ips4o_profile_enable(False)
    mean_ms = statistics.mean(step_ms)
    if ws > 1:
        mean_ms = replica_ms(step_ms, "cuda")
    # verify the last output against the oracle (never report an unverified run)
    ok = ver.check(work.t().contiguous() if kv else work) if ver else None

    # end-to-end: host (pinned) buffer -> device -> sort -> host, through the C ABI
    e2e = None
    if rank == 0 and args.e2e_steps > 0 and not kv:
        h = torch.empty(tuple(work.shape), dtype=work.dtype, pin_memory=True)
        hsrc = pristine.cpu().pin_memory()
        e2e_t = []
        for i in range(args.e2e_steps + 1):
            h.copy_(hsrc)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ips4o.ips4o_sort_host(h.data_ptr(), n, et, sptr)
            dt = time.perf_counter() - t0
            if i > 0:
                e2e_t.append(dt)
        e2e = {"value": n / statistics.mean(e2e_t) / 1e9, "unit": "Gelem/s",
               "h2d_bytes_per_step": n * esize, "d2h_bytes_per_step": n * esize,
               "ms_per_step": statistics.mean(e2e_t) * 1e3, "path": "ips4o_sort_host (pinned host buffer)"}

    if rank != 0:
        if ws > 1:
            torch.distributed.destroy_process_group()
        return 0

    peak, peak_src, peaks = measured_peaks()
    # dominant kernel and its roofline (algorithmic bytes / live event-timed duration)
    kinds = {k: v for k, v in prof.items() if v[0] > 0}
    dom = max(kinds, key=lambda k: kinds[k][1]) if kinds else None
    nl, msk = kinds[dom] if kinds else (1, 0.0)
    dist_el = stats["distributed_elements"]
    base_el = stats["base_elements"]
    per_step_bytes = {
        "classify_flush": 2 * dist_el * esize,   # read every element + flush write
        "block_permute": 2 * dist_el * esize,    # read + write of every block
        "base_case": 2 * base_el * esize,        # read + write once
    }
    launches_per_step = nl / args.steps
    roof = None
    if dom in per_step_bytes:
        bytes_per_launch = per_step_bytes[dom] / launches_per_step
        avg_ms = msk / nl
        achieved = bytes_per_launch / (avg_ms * 1e-3) / 1e9
        traffic = load_traffic(args.config, dom)
        roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                "bytes_per_launch": bytes_per_launch, "avg_launch_ms": avg_ms,
                "share_of_step": msk / max(sum(v[1] for v in kinds.values()), 1e-12),
                "timing": "per-launch CUDA events on the sort stream over a second K-step region "
                          "right after the timed one (same workload)"}
    L = levels_for(n, esize)
    t_roof_nom = 4 * n * esize * L / (BW_NOMINAL * 1e9)
    t_roof_meas = 4 * n * esize * L / (peak * 1e9)
    per_gpu_s = mean_ms * 1e-3
    value = replica_value(n, ws, mean_ms)
    line = {
        "metric": METRIC, "value": value, "unit": "Gelem/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": mean_ms, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": DTYPE[et], "data": "synthetic",
        "config": {"workload": desc, "n": n, "elem_bytes": esize,
                   "parallelism": "replicas" if ws > 1 else "single-gpu",
                   "l2": "input larger than L2 (126 MB) except C1; restored from a pristine device "
                         "copy before every step, outside the events"},
        "roofline": roof,
        "step_roofline": {"levels": L, "bytes": 4 * n * esize * L,
                          "frac_at_8TBs": t_roof_nom / per_gpu_s, "frac_at_measured": t_roof_meas / per_gpu_s},
        "kernels_ms_per_step": {k: v[1] / args.steps for k, v in kinds.items()},
        "gpu_launches": launches,
        "verified": ok,
        "verified_against": "oracle.sort (oracle/, the paper's sequential IS4o), element by element",
        "aux_bytes": stats["aux_bytes"], "aux_frac_of_input": stats["aux_bytes"] / (n * esize),
        "sort_stats": stats,
        "clocks": clk.summary(),
        "ms_per_step_min": min(step_ms), "ms_per_step_median": statistics.median(step_ms),
        "sorted_gbs": n * esize / per_gpu_s / 1e9,
        "step_roofline_with_base": {"bytes": (4 * L + 2) * n * esize,
                                    "frac_at_8TBs": (4 * L + 2) * n * esize / 8.0e12 / per_gpu_s},
    }
    if e2e:
        line["e2e"] = e2e
    if ws == 1 and not args.no_cpu_baseline:
        dist_name = CONFIGS[args.config][0]
        line["cpu_baseline"] = cpu_baseline(dist_name, min(CONFIGS[args.config][1], args.cpu_log2))
        line["cpu_parallel_baseline"] = cpu_parallel_baseline(a, et)
    print(json.dumps(line), flush=True)
    if ws > 1:
        torch.distributed.destroy_process_group()
    return 0 if ok in (True, None) else 1


def replica_ms(step_ms, device) -> float:
    """Replicas only: the job's time per step is the slowest rank's mean step
    time (max over ranks of the device-timed totals); value = all ranks' elements / that."""
    import torch
    t = torch.tensor([sum(step_ms)], device=device, dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item()) / len(step_ms)


def replica_value(n: int, ws: int, mean_ms: float) -> float:
    """Whole-job throughput in Gelem/s: every rank sorts its own n elements per step."""
    return ws * n / (mean_ms * 1e-3) / 1e9


def load_traffic(cfg: str, kernel: str):
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    v = d.get(cfg, {}).get(kernel)
    return v


class OracleVerify:
    """The last timed output is checked against the oracle (BASELINE.md "verify
    before reporting"): the oracle sorts a host copy of the input in a background thread
    (the C oracle releases the GIL) while the GPU is being timed; then the GPU output must
    equal it -- bit for bit for u64/f64 keys; for records, the key sequence bit for bit and
    the record multiset (Pair16: payloads a permutation carrying their original keys)."""

    def __init__(self, a, et):
        import oracle  # test infrastructure: only the verification leg uses it
        self.a, self.et, self.res = a, et, None
        self.thr = threading.Thread(target=lambda: setattr(self, "res", oracle.sort(a)), daemon=True)
        self.thr.start()

    def check(self, work) -> bool:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from gpu_util import to_host
        got = to_host(work, self.et)
        self.thr.join()
        exp, a, et = self.res, self.a, self.et
        if et in (W.ELEM_U64, W.ELEM_F64):
            return bool(np.array_equal(got.view(np.uint64), exp.view(np.uint64)))
        if et in (W.ELEM_PAIR_F64, W.ELEM_QUARTET_F64):
            nk = 1 if et == W.ELEM_PAIR_F64 else 3
            pay = got[:, nk].astype(np.int64)
            return bool(np.array_equal(got[:, :nk].view(np.uint64), exp[:, :nk].view(np.uint64)) and
                        np.array_equal(np.sort(pay), np.arange(a.shape[0])) and
                        np.array_equal(a[pay, :nk].view(np.uint64), got[:, :nk].view(np.uint64)))
        if et == W.ELEM_PAIR:
            # (the Pair16 workload's payload is the original index)
            pay = got[:, 1]
            return bool(np.array_equal(got[:, 0], exp[:, 0]) and
                        np.array_equal(np.sort(pay), np.arange(a.shape[0], dtype=np.uint64)) and
                        np.array_equal(a[pay.astype(np.int64), 0], got[:, 0]))
        if not np.array_equal(got[:, :10], exp[:, :10]):
            return False
        return bool(np.array_equal(np.sort(np.ascontiguousarray(got).view("S100").ravel()),
                                   np.sort(np.ascontiguousarray(exp).view("S100").ravel())))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=15)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="H", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=None, help="override n (debug)")
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-log2", type=int, default=25)
    ap.add_argument("--ref-log2", type=int, default=23)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-kernel-events", action="store_true",
                    help="(diagnostic) skip the per-kernel event region: no roofline line")
    ap.add_argument("--no-verify", action="store_true", help="(diagnostic) skip the oracle check")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # replicas: one process per GPU through torch.distributed.run
        import socket
        with socket.socket() as so:
            so.bind(("127.0.0.1", 0))
            port = so.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
