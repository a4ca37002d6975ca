"""Benchmark of the ChASE hot path on B200: one step = chase_filter (Chebyshev filter, Eq.(1),
P:118-122) + chase_cholqr (Alg.4-selected CholeskyQR variant) on the resident synthetic
workload, through the C-ABI (libchase.so).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2|C3|C4|C5|W|R|auto]
    python bench.py --gpus N ...      (N > 1 without torchrun: re-launches itself under
                                       torch.distributed.run on 127.0.0.1, one rank per GPU)
    python bench.py --impl reference ...                         (CPU oracle arm)

The main series (`value`, BASELINE.json metric) is weak scaling of C2 (N grows with
sqrt(#GPUs), nev = 2250, nex = 750, degree 20; grids 1x1, 2x1, 2x2, 2x4):
    N=1 C2 (N=30000)   N=2 W2 (N=42432)   N=4 W4 (N=60000)   N=8 W8 (N=84848)
Sub-records on the same line (each its own handle, fewer steps):
    strong_c3   C3 (N=60000 complex Clement, n=1300, degree 20) on the same grid: strong scaling
    real        real-symmetric Wilkinson, ramp degrees 10..36 (C5 recipe): N=60000 at 1 GPU,
                84848 / 120000 at 2 / 4 (weak), C5 itself (N=200000) at 8
    target_c4   C4 (N=120000 complex Uniform, n=1600, 2x4) at N=8: the north-star target
N > 1 filter steps run as fused HEMM + NVLink peer-memory reduction kernels (--comm fused,
default) or as HEMM + ncclAllReduce (--comm nccl).
Metric: algorithmic filter flops 8 N^2 sum_j d_j (complex; 2 N^2 sum d real) divided by the whole
step time (filter + QR), max over ranks -- QR time is charged against the filter number.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import math
import os
import socket
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "Chebyshev filter FP64 TFLOP/s (max over ranks) at 1/2/4/8 B200; % of FP64 peak"
# FP64 tensor (DMMA) peak measured on this pool's B200 by tools/microbench/fp64_peak.cu
# (profiles/r01/fp64_peak.log: 37.1 TFLOP/s burst and sustained at 1965 MHz).
# MEASURED_PEAKS.json carries no FP64 figure.
FP64_PEAK_TFLOPS = 37.1
GRIDS = {1: (1, 1), 2: (2, 1), 4: (2, 2), 8: (2, 4)}
SERIES_FILE = "/tmp/chase_bench_series.json"    # N=1 results of this box, for efficiency_vs_n1


def workload(n_gpus: int, name: str):
    import chase_inputs as ci
    if name == "auto":
        name = "C2" if n_gpus == 1 else "W"
    if name == "W":   # weak-scaling point of C2 (N grows with sqrt(#GPUs))
        N = 16 * int(round(30000 * math.sqrt(n_gpus) / 16))    # multiple of 16: 3D TMA path
        return dict(name=f"W{n_gpus}", N=N, nev=2250, nex=750, complex_=True, spectrum="uniform",
                    seed=2, degree=20,
                    desc=f"C2 weak-scaling point: N={N} complex Hermitian Uniform, nev=2250 nex=750, "
                         f"degree 20")
    if name == "R":   # real Wilkinson weak series (C5 recipe), C5 itself at 8 GPUs
        if n_gpus == 8:
            name = "C5"
        else:
            N = 16 * int(round(60000 * math.sqrt(n_gpus) / 16))
            return dict(name=f"R{n_gpus}", N=N, nev=2000, nex=500, complex_=False,
                        spectrum="wilkinson", seed=5, degree=None,
                        desc=f"C5 recipe at N={N}: real symmetric Wilkinson, nev=2000 nex=500, "
                             f"ramp degrees 10-36")
    c = ci.CONFIGS[name]
    deg = "ramp 10-36" if c.degree is None else f"degree {c.degree}"
    return dict(name=name, N=c.N, nev=c.nev, nex=c.nex, complex_=c.complex_, spectrum=c.spectrum,
                seed=c.seed, degree=c.degree,
                desc=f"{name}: N={c.N} {'complex Hermitian' if c.complex_ else 'real symmetric'} "
                     f"{c.spectrum.capitalize()}, nev={c.nev} nex={c.nex}, {deg}")


def spectrum(w):
    import chase_inputs as ci
    if w["spectrum"] == "uniform":
        return ci.uniform_spectrum(w["N"])
    if w["spectrum"] == "clement":
        return ci.clement_spectrum(w["N"])
    return ci.wilkinson_spectrum(w["N"])


def degrees_of(w):
    import chase_inputs as ci
    n = w["nev"] + w["nex"]
    return ci.uniform_degrees(n, w["degree"]) if w["degree"] else ci.ramp_degrees(n)


def generator(w, lam):
    import chase_inputs as ci
    return ci.dft_phase(lam, w["seed"]) if w["complex_"] else ci.hartley_sign(lam, w["seed"])


def filter_flops(w, degrees):
    return (8.0 if w["complex_"] else 2.0) * float(w["N"]) ** 2 * float(np.sum(degrees))


def qr_flops_per_gpu(w, n, passes, p):
    """Per GPU per pass: Gram (upper half, 4 (N/p) n^2 real flops complex) + TRSM (4 (N/p) n^2)
    on the rank's N/p rows, + POTRF (4 n^3 / 3), which every rank repeats."""
    f = 8.0 * (w["N"] / p) * n * n + 4.0 * n ** 3 / 3.0
    return passes * (f if w["complex_"] else f / 4.0)


def src_hash():
    """Hash of the GEMM kernel sources: a committed ncu traffic figure is used only for them."""
    h = hashlib.sha256()
    for f in ("common.cuh", "zgemm.cuh", "dgemm.cuh", "gemm_tail.cuh"):
        with open(os.path.join(ROOT, "paper_2309_15595_b200", "csrc", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


class Clocks:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"bench_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                          "-lms", "200", "-i", str(self.index)], stdout=self.f,
                                         stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.f.close()
        sm, mx, pw, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
                pw.append(float(parts[3]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": max(mx), "power_w_max": max(pw),
                "samples": len(sm), "reasons": sorted(reasons)}


class NvLink:
    """NVLink data bytes moved by this GPU, summed over its active links, read around the timed
    region (the fused kernel's peer traffic).  NVML field values: COUNT_XMIT/RCV_BYTES (bytes;
    the Blackwell counters), else THROUGHPUT_DATA_TX/RX (KiB)."""

    def __init__(self, index: int):
        self.index = index
        self.h, self.err, self.links = None, None, []
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            for l in range(18):
                try:
                    if pynvml.nvmlDeviceGetNvLinkState(self.h, l) == 1:
                        self.links.append(l)
                except Exception:
                    pass
            if not self.links:
                self.err = "no active NVLink reported by NVML"
        except Exception as exc:
            self.h, self.err = None, f"NVML: {exc}"

    def read(self):
        if self.h is None or not self.links:
            return self._smi()
        nv = self.nv
        for tx_id, rx_id, scale, name in (
                (getattr(nv, "NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES", None),
                 getattr(nv, "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES", None), 1, "COUNT_XMIT/RCV_BYTES"),
                (nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, nv.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 1024,
                 "THROUGHPUT_DATA_TX/RX")):
            if tx_id is None:
                continue
            try:
                tx = rx = 0
                ok = True
                for l in self.links:
                    vals = nv.nvmlDeviceGetFieldValues(self.h, [(tx_id, l), (rx_id, l)])
                    if vals[0].nvmlReturn != 0 or vals[1].nvmlReturn != 0:
                        ok = False
                        self.err = f"{name}: nvmlReturn {vals[0].nvmlReturn}/{vals[1].nvmlReturn}"
                        break
                    tx += vals[0].value.ullVal
                    rx += vals[1].value.ullVal
                if ok:
                    self.field = name
                    return scale * tx, scale * rx
            except Exception as exc:
                self.err = f"{name}: {exc}"
        return self._smi()

    def _smi(self):
        """Fallback: `nvidia-smi nvlink -gt d` (per-link data Tx/Rx KiB counters)."""
        try:
            out = subprocess.run(["nvidia-smi", "nvlink", "-gt", "d", "-i", str(self.index)],
                                 capture_output=True, text=True, timeout=20).stdout
            tx = rx = 0
            seen = False
            for line in out.splitlines():
                parts = line.replace(":", " ").split()
                if "Tx" in parts and "KiB" in parts:
                    tx += int(parts[parts.index("KiB") - 1]); seen = True
                elif "Rx" in parts and "KiB" in parts:
                    rx += int(parts[parts.index("KiB") - 1]); seen = True
            if seen:
                self.field = "nvidia-smi nvlink -gt d"
                return 1024 * tx, 1024 * rx
            self.err = (self.err or "") + f"; nvidia-smi nvlink -gt d: no counters ({out.strip()[:80]!r})"
        except Exception as exc:
            self.err = (self.err or "") + f"; nvidia-smi nvlink: {exc}"
        return None


def cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


# ====================================================================== CPU oracle (baseline)
def oracle_sample(A_host, V0_host, degrees, b, cols):
    """Time the triple-loop C++ oracle filter (oracle/cpp/chase_oracle.cpp, as it stands; OpenMP
    over all host cores) on `cols` columns of the same workload (full A).  Returns (s, flops)."""
    from oracle import cpp_oracle
    cpp_oracle.load()
    V = np.asfortranarray(V0_host[:, :cols])
    d = list(int(x) for x in degrees[:cols])
    t0 = time.perf_counter()
    cpp_oracle.filter(A_host, V, d, b.c, b.e, b.mu_1)
    t = time.perf_counter() - t0
    N = A_host.shape[0]
    return t, (8.0 if np.iscomplexobj(A_host) else 2.0) * N * N * sum(d)


def run_reference(args):
    """--impl reference: the CPU oracle on the box's host cores, on a bounded sample of the
    same workload (one column of V per step, full degree, full A)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import torch
    import chase_inputs as ci
    n_gpus = args.gpus
    w = workload(n_gpus, args.config)
    if w["N"] > 60000:
        print(json.dumps({"impl": "reference", "unavailable":
                          f"the CPU oracle needs the full {w['N']}^2 matrix in host memory "
                          f"({16 * w['N'] ** 2 / 1e9:.0f} GB > host RAM)"}))
        return
    lam = spectrum(w)
    n = w["nev"] + w["nex"]
    degrees = degrees_of(w)
    b = ci.bounds_from_spectrum(lam, n)
    gen = generator(w, lam)
    torch.set_num_threads(cores())
    A = gen.block(0, w["N"], 0, w["N"], device="cpu").numpy().T      # host, column-major
    V0 = ci.gaussian_block(w["N"], n, w["seed"] + 1000, w["complex_"])
    # bounded sample: one column, degree 20 up to N = 30000, degree 4 above (each matvec streams
    # the whole 16 N^2-byte matrix), so the W + K steps stay within a few minutes
    d_sample = np.array([int(degrees[0]) if w["N"] <= 30000 else 4], dtype=np.int32)
    for _ in range(args.warmup):
        oracle_sample(A, V0, d_sample, b, 1)
    ts, fl = [], 0.0
    for _ in range(args.steps):
        t, f = oracle_sample(A, V0, d_sample, b, 1)
        ts.append(t)
        fl += f
    tot = sum(ts)
    value = fl / tot / 1e12
    sample = (f"triple-loop C++ oracle filter (oracle/cpp) on 1 of {n} columns per step (degree "
              f"{int(d_sample[0])}), full {w['N']}x{w['N']} A, OpenMP over {cores()} host cores")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": n_gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": w["desc"], "sample": sample},
        "cpu_baseline": {"value": value, "unit": "TFLOP/s", "cores": cores(), "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": value, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


# ====================================================================== GPU arm
class Ctx:
    """Per-process state: rank, grid, device, stream, process group."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.torch, self.dist = torch, dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world != args.gpus:
            raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={self.world}")
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.world > 1:
            dist.init_process_group("nccl", device_id=self.dev)
        self.p, self.q = GRIDS[self.world]
        self.myrow, self.mycol = self.rank // self.q, self.rank % self.q
        self.stream = torch.cuda.current_stream(self.dev)
        self.args = args

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()
        self.torch.cuda.synchronize()

    def allmax(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def allsum(self, x):
        if self.world == 1:
            return x
        t = self.torch.tensor([x], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t)
        return float(t.item())


class Problem:
    """One workload resident on this rank: handle (+ fused region), A_local, V0 (pinned host and
    device copies)."""

    def __init__(self, cx: Ctx, w, comm: str):
        import chase_inputs as ci
        import paper_2309_15595_b200 as cb
        torch = cx.torch
        self.cx, self.w, self.cb = cx, w, cb
        self.N, self.n = w["N"], w["nev"] + w["nex"]
        self.lam = spectrum(w)
        self.degrees = degrees_of(w)
        self.b = ci.bounds_from_spectrum(self.lam, self.n)
        self.bounds = (self.b.mu_1, self.b.mu_ne, self.b.b_sup)
        self.est = cb.chase_cond_est(self.lam, self.b.c, self.b.e, self.degrees, 0)
        dtype = cb.CHASE_C128 if w["complex_"] else cb.CHASE_R64
        uid = None
        if cx.world > 1:
            from paper_2309_15595_b200 import dist as cdist
            uid = cdist.share_unique_id(cb.chase_get_unique_id)
        self.h = cb.Chase(dtype, self.N, self.n, cx.p, cx.q, cx.myrow, cx.mycol, uid, cx.local, cx.stream)
        self.comm_mode = "none"
        if cx.world > 1:
            self.comm_mode = "nccl"
            if comm == "fused":
                from paper_2309_15595_b200 import dist as cdist
                try:
                    cdist.enable_fused_comm(self.h)
                    self.comm_mode = "fused HEMM + NVLink peer-memory reduction"
                except Exception as exc:      # e.g. no peer mapping on this box: stay on NCCL
                    self.comm_mode = f"nccl (fused unavailable: {type(exc).__name__})"
        h = self.h
        gen = generator(w, self.lam)
        self.A_t = gen.block(h.r0, h.n_r, h.c0, h.n_c, device=cx.dev)     # (n_c, n_r) storage
        self.A_local = self.A_t.T                                         # column-major n_r x n_c
        V0_full = ci.gaussian_block(self.N, self.n, w["seed"] + 1000, w["complex_"])
        self.V0_rows = np.asfortranarray(V0_full[h.r0:h.r0 + h.n_r])
        del V0_full
        self.V0_host = torch.from_numpy(np.ascontiguousarray(self.V0_rows.T)).pin_memory()
        self.V_t = self.V0_host.to(cx.dev)                                # (n, n_r) storage
        self.V = self.V_t.T
        self.F = filter_flops(w, self.degrees)
        torch.cuda.synchronize()

    def step(self, V=None, ev=None):
        V = self.V if V is None else V
        self.h.filter(self.A_local, V, self.degrees, self.b.c, self.b.e, self.bounds)
        if ev is not None:
            ev.record(self.cx.stream)
        return self.h.cholqr(V, self.est)

    def close(self):
        self.h.close()
        for k in ("A_t", "A_local", "V_t", "V", "V0_host"):
            setattr(self, k, None)
        self.cx.torch.cuda.synchronize()
        self.cx.torch.cuda.empty_cache()


def timed_run(cx: Ctx, P: Problem, steps: int, warmup: int, clocks=None, nvlink=None):
    """W untimed warm-up steps, then K steps bracketed by barrier + synchronize; CUDA events on
    the handle's stream split each step into filter and QR.  Max over ranks."""
    torch, cb = cx.torch, P.cb
    qr_info = None
    cx.barrier()                                      # no rank starts the fused protocol early
    for _ in range(warmup):
        qr_info = P.step()
    cx.barrier()
    cb.chase_profile_enable(P.h.h, True)
    cb.chase_profile_read(P.h.h)                      # reset counters
    if clocks:
        clocks.start()
    nv0 = nvlink.read() if nvlink else None
    cx.barrier()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for k in range(steps):
        ev[k][0].record(cx.stream)
        qr_info = P.step(ev=ev[k][1])
        ev[k][2].record(cx.stream)
    cx.barrier()
    nv1 = nvlink.read() if nvlink else None
    clk = clocks.stop() if clocks else None
    total = ev[0][0].elapsed_time(ev[-1][2])
    filt = sum(e[0].elapsed_time(e[1]) for e in ev)
    qr = sum(e[1].elapsed_time(e[2]) for e in ev)
    prof_ms, prof_n = cb.chase_profile_read(P.h.h)
    cb.chase_profile_enable(P.h.h, False)
    hemm_local = prof_ms["hemm"]
    res = dict(ms=cx.allmax(total), filter_ms=cx.allmax(filt), qr_ms=cx.allmax(qr),
               hemm_ms=cx.allmax(hemm_local), prof_ms=prof_ms, prof_n=prof_n, qr_info=qr_info, clocks=clk)
    if nv0 is not None and nv1 is not None:
        res["nvlink_tx"] = cx.allsum(nv1[0] - nv0[0])
        res["nvlink_rx"] = cx.allsum(nv1[1] - nv0[1])
    return res


def hemm_roofline(cx: Ctx, P: Problem, r, steps):
    """achieved = per-launch algorithmic HEMM flops / mean launch time (library CUDA events)."""
    D = int(np.max(P.degrees))
    per_gpu = P.F / cx.world
    avg_ms = r["hemm_ms"] / (steps * D)
    achieved = per_gpu / D / (avg_ms / 1e3) / 1e12
    return dict(achieved=achieved, frac=achieved / FP64_PEAK_TFLOPS, per_launch_flops=per_gpu / D,
                avg_launch_ms=avg_ms)


def fused_nvlink_bytes(cx: Ctx, P: Problem):
    """Algorithmic NVLink bytes of one filter call, all ranks: per step with an m-member
    communicator each rank pushes (m-1)/m of its partial output block to the tile owners and
    broadcasts its 1/m of owned tiles to m-1 members: 2 (m-1)/m rows_out k esize."""
    import chase_inputs as ci
    es = 16 if P.w["complex_"] else 8
    tot = 0.0
    for rank in range(cx.world):
        i, j = rank // cx.q, rank % cx.q
        n_r, n_c, _, _ = ci.block_dims(P.N, cx.p, cx.q, i, j)
        for s in range(1, int(np.max(P.degrees)) + 1):
            k = int(np.sum(P.degrees >= s))
            m, rows = (cx.p, n_c) if s % 2 == 1 else (cx.q, n_r)
            if m > 1:
                tot += 2.0 * (m - 1) / m * rows * k * es
    return tot


def series_file(update=None):
    try:
        d = json.load(open(SERIES_FILE))
    except Exception:
        d = {}
    if update:
        d.update(update)
        with open(SERIES_FILE, "w") as f:
            json.dump(d, f)
    return d


def sub_record(cx: Ctx, name: str, comm: str, steps: int = 2, warmup: int = 1):
    """A secondary workload on the same grid (own handle): throughput, per-GPU rate, HEMM roofline
    fraction; efficiency against this box's N=1 run of the same record when one was made."""
    w = workload(cx.world, name)
    P = Problem(cx, w, comm)
    r = timed_run(cx, P, steps, warmup)
    rf = hemm_roofline(cx, P, r, steps)
    value = P.F * steps / (r["ms"] / 1e3) / 1e12
    out = {"workload": w["desc"], "grid": f"{cx.p}x{cx.q}", "value": value, "unit": "TFLOP/s",
           "per_gpu_tflops": value / cx.world, "pct_of_fp64_peak_per_gpu": 100 * value / cx.world / FP64_PEAK_TFLOPS,
           "ms_per_step": r["ms"] / steps, "filter_ms_per_step": r["filter_ms"] / steps,
           "qr_ms_per_step": r["qr_ms"] / steps, "qr_variant": r["qr_info"]["variant"],
           "steps": steps, "warmup": warmup,
           "roofline": {"bound": "tensor", "kernel": ("zgemm" if w["complex_"] else "dgemm") +
                        ("_fused_kernel" if "fused" in P.comm_mode else "_kernel"),
                        "achieved": rf["achieved"], "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                        "frac": rf["frac"]},
           "filter_comm": P.comm_mode}
    P.close()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="auto")
    ap.add_argument("--impl", default="native", choices=["native", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip RR / residuals / HHQR comparison")
    ap.add_argument("--no-sub", action="store_true", help="skip the strong_c3 / real / target_c4 sub-records")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-cols", type=int, default=2)
    ap.add_argument("--comm", default="fused", choices=["fused", "nccl"],
                    help="N > 1: filter steps as fused HEMM + NVLink reduction kernels, or HEMM + ncclAllReduce")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torch.distributed.run on this node
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
        s.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__),
               *sys.argv[1:]]
        return subprocess.call(cmd)
    if args.impl == "reference":
        return run_reference(args)

    cx = Ctx(args)
    torch = cx.torch
    import paper_2309_15595_b200 as cb

    w = workload(cx.world, args.config)
    P = Problem(cx, w, args.comm)
    n_gpus, N, n = cx.world, P.N, P.n
    clocks = Clocks(cx.local)
    nvlink = NvLink(cx.local) if "fused" in P.comm_mode else None
    r = timed_run(cx, P, args.steps, args.warmup, clocks, nvlink)
    ms = r["ms"]
    F = P.F
    value = F * args.steps / (ms / 1e3) / 1e12
    rf = hemm_roofline(cx, P, r, args.steps)
    gpu_launches = int(sum(r["prof_n"][k] for k in ("hemm", "gram", "potrf", "trsm", "other", "hhqr")))
    stream, e0, e1 = cx.stream, torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    extras = {}

    if not args.no_extras:
        # ---- NEXT-2: Rayleigh-Ritz (Alg.2 l.16-22) on the step's orthonormal output, timed once
        cx.barrier()
        cb.chase_profile_enable(P.h.h, True)
        cb.chase_profile_read(P.h.h)
        e0.record(stream)
        ritz, rr_levels = P.h.rayleigh_ritz(P.A_local, P.V)
        e1.record(stream)
        cx.barrier()
        rr_prof, _ = cb.chase_profile_read(P.h.h)
        cb.chase_profile_enable(P.h.h, False)
        lam_sorted = np.sort(P.lam)
        extras["rayleigh_ritz"] = {
            "ms": cx.allmax(e0.elapsed_time(e1)), "eigensolver_ms": cx.allmax(rr_prof["other"]),
            "hemm_ms": cx.allmax(rr_prof["hemm"]), "dc_levels": rr_levels,
            "max_ritz_minus_eig_lowest_nev": float(np.max(ritz[:w["nev"]] - lam_sorted[:w["nev"]])),
            "note": "chase_rayleigh_ritz on the step output (NEXT-2): B = H C (one HEMM), the quotient, "
                    "own HEEVD (Householder tridiagonalisation + divide and conquer + back-transform), "
                    "V <- V Y; not part of the step"}
        # ---- NEXT-1: residual norms (Alg.2 l.23-28) of the Ritz pairs, timed separately
        P.h.residuals(P.A_local, P.V, ritz)                     # warm-up
        cx.barrier()
        e0.record(stream)
        resid = P.h.residuals(P.A_local, P.V, ritz)
        e1.record(stream)
        cx.barrier()
        res_ms = cx.allmax(e0.elapsed_time(e1))
        extras["residuals"] = {
            "ms": res_ms, "unit": "TFLOP/s",
            "tflops": (8.0 if w["complex_"] else 2.0) * float(N) ** 2 * n / (res_ms / 1e3) / 1e12,
            "max_resid": float(np.max(resid)),
            "note": "chase_residuals on the step output (NEXT-1, Alg.2 l.23-28), not part of the step"}
        # ---- CholeskyQR (Alg.4) vs Householder QR (Alg.4 l.9 / the HHQR mode of P:448, Table 3)
        P.V_t.copy_(P.V0_host)
        P.h.filter(P.A_local, P.V, P.degrees, P.b.c, P.b.e, P.bounds)
        Xf_t = P.V_t.clone()
        qr_cmp = {}
        for name, fn in (("cholqr", lambda: P.h.cholqr(P.V, P.est)), ("hhqr", lambda: P.h.hhqr(P.V))):
            P.V_t.copy_(Xf_t)
            fn()                                           # warm-up
            P.V_t.copy_(Xf_t)
            cx.barrier()
            e0.record(stream)
            fn()
            e1.record(stream)
            cx.barrier()
            qr_cmp[name + "_ms"] = cx.allmax(e0.elapsed_time(e1))
        del Xf_t
        qr_cmp["cholqr_speedup_over_hhqr"] = qr_cmp["hhqr_ms"] / qr_cmp["cholqr_ms"]
        qr_cmp["note"] = ("same filtered block; paper Table 3 (P:455-483) compares ChASE with HHQR "
                          "(ScaLAPACK, CPU) against CholeskyQR; here both run on the GPU")
        extras["qr_vs_hhqr"] = qr_cmp

    # ---- end-to-end through the public API with host buffers: every step's V is copied in from
    # pinned host memory and its result copied back out, double-buffered like a production caller
    # (step k+1's H2D and step k's D2H on a copy stream under the compute).
    e2e = None
    if not args.no_e2e:
        out_host = torch.empty_like(P.V0_host).pin_memory()
        bufs = [P.V_t, torch.empty_like(P.V_t)]
        cstream = torch.cuda.Stream(cx.dev)
        ev_in = [torch.cuda.Event() for _ in range(args.steps)]
        ev_done = [torch.cuda.Event() for _ in range(args.steps)]
        ev_out = torch.cuda.Event()
        cx.barrier()
        e0.record(stream)
        cstream.wait_stream(stream)
        with torch.cuda.stream(cstream):
            bufs[0].copy_(P.V0_host, non_blocking=True)
            ev_in[0].record(cstream)
        for k in range(args.steps):
            vb = bufs[k % 2]
            stream.wait_event(ev_in[k])
            P.step(vb.T)
            ev_done[k].record(stream)
            with torch.cuda.stream(cstream):
                if k + 1 < args.steps:
                    bufs[(k + 1) % 2].copy_(P.V0_host, non_blocking=True)
                    ev_in[k + 1].record(cstream)
                cstream.wait_event(ev_done[k])
                out_host.copy_(vb, non_blocking=True)
        ev_out.record(cstream)
        stream.wait_event(ev_out)
        e1.record(stream)
        cx.barrier()
        e2e_ms = cx.allmax(e0.elapsed_time(e1))
        del bufs
        nbytes = P.V0_host.numel() * P.V0_host.element_size()
        e2e = {"value": F * args.steps / (e2e_ms / 1e3) / 1e12, "unit": "TFLOP/s",
               "ms_per_step": e2e_ms / args.steps, "h2d_bytes_per_step": int(nbytes),
               "d2h_bytes_per_step": int(nbytes),
               "note": "A_local resident (set once, as the paper distributes H once); V copied in from "
                       "pinned host memory and the result out every step, double-buffered on a copy "
                       "stream (step k+1 in and step k out overlap compute); per-rank bytes"}

    # ---- CPU oracle baseline on a bounded sample of the same workload (rank 0, N=1)
    cpu = None
    if cx.rank == 0 and n_gpus == 1 and not args.no_cpu_baseline:
        torch.set_num_threads(cores())
        A_host = P.A_t.cpu().numpy().T                   # same bits the GPU used
        t, fl = oracle_sample(A_host, np.asfortranarray(P.V0_rows), P.degrees, P.b, args.cpu_cols)
        cpu = {"value": fl / t / 1e12, "unit": "TFLOP/s", "cores": cores(), "kind": "oracle",
               "sample": f"triple-loop C++ oracle filter (oracle/cpp) on {args.cpu_cols} of {n} columns "
                         f"(degree {int(P.degrees[0])}), full {N}x{N} A copied from the device, {t:.1f} s"}
        del A_host

    nvl = None
    if nvlink is not None and "nvlink_tx" not in r:
        nvl = {"unavailable": nvlink.err}
    if "nvlink_tx" in r:
        alg = fused_nvlink_bytes(cx, P) * args.steps
        nvl = {"counter": nvlink.field, "tx_bytes_all_ranks": r["nvlink_tx"], "rx_bytes_all_ranks": r["nvlink_rx"],
               "algorithmic_bytes_all_ranks": alg,
               "tx_over_algorithmic": r["nvlink_tx"] / alg if alg else None,
               "note": "NVML NVLink data counters around the timed steps (filter + QR: the QR's Gram "
                       "AllReduce is NCCL traffic too); algorithmic = fused filter pushes + broadcasts"}
    comm_mode = P.comm_mode
    P.close()

    # ---- sub-records (own handles, fewer steps)
    subs = {}
    if not args.no_sub:
        subs["strong_c3"] = sub_record(cx, "C3", args.comm)
        subs["real"] = sub_record(cx, "R", args.comm)
        if n_gpus == 8:
            subs["target_c4"] = sub_record(cx, "C4", args.comm)

    # ---- efficiency against this box's N=1 run (same series), when one was made
    eff = {}
    if cx.rank == 0:
        mine = {"main": {"workload": w["name"], "value": value}}
        for k, v in subs.items():
            mine[k] = {"workload": v["workload"], "value": v["value"], "ms_per_step": v["ms_per_step"]}
        if n_gpus == 1:
            series_file({"n1": mine})
        ref1 = series_file().get("n1")
        if ref1:
            eff["main_weak"] = (value / n_gpus) / ref1["main"]["value"]
            if "strong_c3" in subs and "strong_c3" in ref1:
                eff["strong_c3"] = ref1["strong_c3"]["ms_per_step"] / (n_gpus * subs["strong_c3"]["ms_per_step"])
            if "real" in subs and "real" in ref1:
                eff["real_weak_per_gpu_tflops"] = subs["real"]["per_gpu_tflops"] / ref1["real"]["value"]
        for k in subs:
            if k in eff:
                subs[k]["efficiency_vs_n1"] = eff[k]
        if "real" in subs and "real_weak_per_gpu_tflops" in eff:
            subs["real"]["efficiency_vs_n1"] = eff["real_weak_per_gpu_tflops"]

    traffic = None
    tpath = os.path.join(ROOT, "profiles", "hemm_traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            if tj.get("workload") == w["name"] and tj.get("src_hash") == src_hash():
                traffic = tj.get("bytes_per_launch")
        except Exception:
            traffic = None

    if cx.rank == 0:
        qi = r["qr_info"]
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": n_gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": w["desc"], "grid": f"{cx.p}x{cx.q}", "N": N, "n": n,
                       "sum_degrees": int(np.sum(P.degrees)),
                       "step": "chase_filter + chase_cholqr (Alg.4 variant from Alg.5 estimate)",
                       "l2": "no flush needed: A_local is larger than the 126 MB L2 "
                             f"({(16 if w['complex_'] else 8) * N * N / n_gpus / 1e9:.1f} GB per GPU)",
                       "parallelism": f"2D block grid {cx.p}x{cx.q}",
                       "series": "weak scaling of C2: N = 30000 sqrt(#GPUs), n = 3000, degree 20 (P:545-549)",
                       "filter_comm": comm_mode},
            "pct_of_fp64_peak_per_gpu": 100.0 * value / n_gpus / FP64_PEAK_TFLOPS,
            "efficiency_vs_n1": eff.get("main_weak"),
            "filter_only_tflops": F * args.steps / (r["filter_ms"] / 1e3) / 1e12,
            "qr": {"variant": qi["variant"], "passes": qi["passes"],
                   "ms_per_step": r["qr_ms"] / args.steps, "cond_est": P.est,
                   "tflops_per_gpu": qr_flops_per_gpu(w, n, qi["passes"], cx.p) * args.steps /
                                     max(1e-9, r["qr_ms"] / 1e3) / 1e12,
                   "note": "timed with CUDA events between the end of chase_filter and the end of "
                           "chase_cholqr; flops per GPU = passes x (8 (N/p) n^2 + 4 n^3/3)"},
            "roofline": {"bound": "tensor", "kernel": ("zgemm" if w["complex_"] else "dgemm") +
                         ("_fused_kernel (HEMM + reduction)" if "fused" in comm_mode else "_kernel (HEMM step)"),
                         "achieved": rf["achieved"], "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                         "frac": rf["frac"], "traffic": traffic,
                         "peak_source": "measured FP64 DMMA microbenchmark (profiles/r01/fp64_peak.log); "
                                        "MEASURED_PEAKS.json has no FP64 entry",
                         "per_launch_flops": rf["per_launch_flops"], "avg_launch_ms": rf["avg_launch_ms"]},
            "profile_ms_per_step": {k: v / args.steps for k, v in r["prof_ms"].items()},
            "gpu_launches": gpu_launches,
            **extras,
            "nvlink": nvl,
            **subs,
            "clocks": r["clocks"],
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if cx.world > 1:
        cx.dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
