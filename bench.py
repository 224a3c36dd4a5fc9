"""Benchmark: quantized inverse-operator applies/s and achieved HBM GB/s.

BASELINE.json metric: "inverse-operator applies/sec and achieved HBM GB/s
(frac of roofline) at N=128^2" — config 4 (variable-eps, non-uniform
128x128 grid, N=16384, 5 decimal digits, single fp32 right-hand side).

A step is one apply y = L_eps^-1 rho of the quantized operator resident in
HBM (one K2 launch; plus the NCCL all-gather of the row shards for N>1).
Inputs are larger than L2 (the 3-byte codes of config 4 are 805 MB), so no
L2 flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4]
    python bench.py --impl reference ...   # the reference's CPU kernel

Under torchrun each rank owns a contiguous row block of L^-1 (built on its
own GPU by the block-LU constructor), applies it to rho, and the row blocks
are all-gathered. Rank 0 prints one JSON line.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "inverse-operator applies/sec and achieved HBM GB/s (frac of roofline) at N=128²"
UNIT = "applies/s"
L2_BYTES = 128 * 2**20          # B200 L2 is 126 MB; rounded up


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """Polls NVML every ~10 ms while the timed region runs."""

    def __init__(self, device_index: int):
        self.samples = []
        self.reasons = set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._ok = False
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self._ok = True
        except Exception as e:  # noqa: BLE001
            self.error = str(e)

    _REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
        0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
        0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                for bit, name in self._REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:  # noqa: BLE001
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self._ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self._ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self._ok:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvml unavailable"]}
        return {
            "sm_mhz": statistics.median(self.samples) if self.samples else None,
            "sm_max_mhz": self.max_mhz,
            "reasons": sorted(self.reasons),
            "samples": len(self.samples),
        }


# ------------------------------------------------------------------ dist
def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        backend = "nccl" if args.impl == "ours" else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


# ------------------------------------------------------------------ cpu baseline
def reference_sample(cfg, max_seconds: float, target_step_s: float = 0.25, seed_cols: int = 7):
    """Bounded sample of the workload for the reference CPU kernel: a set of
    C columns of the quantized L^-1 (from a host sparse LU, quantized with the
    reference's rounding), its plan tables (reference build_plan restated),
    and the reference's own compiled plan_apply (oracle/_ref) — or the
    oracle's C port of it when oracle/_ref was not built."""
    from oracle import invop_oracle as O
    import scipy.sparse.linalg as spla

    st = cfg.operator()
    N = st.n
    ref = O.reference_native()
    kind = "reference" if ref is not None else "port"
    # pick the column count so that one sampled apply takes ~target_step_s
    cols = 256
    rng = np.random.default_rng(seed_cols)
    lu = spla.splu(st.to_sparse().tocsc())

    def make(cols):
        J = np.sort(rng.choice(N, size=cols, replace=False))
        E = np.zeros((N, cols))
        E[J, np.arange(cols)] = 1.0
        Z = lu.solve(E)                        # columns J of L^-1
        mant = O.quantize(Z, cfg.digits)       # N x cols
        plan = O.build_plan_rect(mant, cfg.digits)
        return J, plan

    x_full = cfg.rhs()[0]

    def run(J, plan):
        out = np.zeros(N)
        t0 = time.perf_counter()
        if ref is not None:
            ref.plan_apply(plan["col_ptr"], plan["group_coeff"], plan["group_ptr"],
                           plan["entry_rows"], plan["entry_signs"], np.ascontiguousarray(x_full[J]), out)
        else:
            O.plan_apply(plan, x_full[J])
        return time.perf_counter() - t0

    J, plan = make(cols)
    t = run(J, plan)
    scale = max(0.05, min(16.0, target_step_s / max(t, 1e-6)))
    cols = int(min(N, max(16, cols * scale)))
    J, plan = make(cols)
    return dict(J=J, plan=plan, run=run, cols=cols, N=N, kind=kind)


def cpu_baseline(cfg, budget_s: float = 15.0):
    s = reference_sample(cfg, budget_s)
    times = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end or len(times) < 3:
        times.append(s["run"](s["J"], s["plan"]))
        if len(times) >= 50:
            break
    best = min(times)
    per_apply = best * s["N"] / s["cols"]
    return {
        "value": 1.0 / per_apply,
        "unit": UNIT,
        "cores": 1,
        "kind": s["kind"],
        "sample": "%d of %d columns of the quantized L^-1 (all %d rows), reference plan_apply "
                  "best of %d runs, scaled by N/cols; single-threaded (the reference holds the GIL)"
                  % (s["cols"], s["N"], s["N"], len(times)),
        "host_cpus": os.cpu_count(),
        "affinity_cpus": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None,
    }


# ------------------------------------------------------------------ reference arm
def run_reference(args, world, rank):
    from paper_1602_00001_b200 import configs

    if rank != 0:
        return
    cfg = configs.get(args.config)
    # size each step so the whole --steps/--warmup run stays around a minute
    target = max(0.005, min(0.2, 60.0 / max(1, args.steps + args.warmup)))
    s = reference_sample(cfg, 0.0, target_step_s=target)
    for _ in range(args.warmup):
        s["run"](s["J"], s["plan"])
    t0 = time.perf_counter()
    for _ in range(args.steps):
        s["run"](s["J"], s["plan"])
    el = time.perf_counter() - t0
    per_apply = el / args.steps * s["N"] / s["cols"]
    value = 1.0 / per_apply
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_apply * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded; BASELINE.json config %d)" % cfg.key,
        "config": {"workload": cfg.name, "N": cfg.N, "digits": cfg.digits, "nrhs": 1},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": s["kind"],
                         "sample": "%d of %d columns per step, scaled by N/cols" % (s["cols"], s["N"])},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def run_ours(args, world, rank, local):
    import torch

    import paper_1602_00001_b200 as invop
    from paper_1602_00001_b200 import configs, _lib as L

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    cfg = configs.get(args.config)
    st = cfg.operator()
    N = st.n
    rows = N // world
    row0 = rank * rows
    if rank == world - 1:
        rows = N - row0
    # ---- setup (timed separately): block-LU factor + construct + encode
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dop = invop.DeviceOperator(st).factor()
    torch.cuda.synchronize()
    t_factor = time.perf_counter() - t0
    plan = dop.quantized_rows(cfg.digits, row0, rows)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0

    X = cfg.rhs()
    if args.nrhs:
        reps = -(-args.nrhs // X.shape[0])
        X = np.ascontiguousarray(np.tile(X, (reps, 1))[:args.nrhs])
    k = X.shape[0]
    x64 = torch.tensor(X, dtype=torch.float64, device=dev)      # [k, N]
    x32 = x64.float().contiguous()
    y32 = torch.empty((k, rows), dtype=torch.float32, device=dev)
    full = torch.empty((world, k, rows), dtype=torch.float32, device=dev) if world > 1 else None
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    h = plan.handle
    import ctypes as C

    def launch_fast():
        L.lib.invop_apply(h, x32.data_ptr(), N, y32.data_ptr(), rows, k, L.F32, L.MODE_FAST,
                          C.c_void_p(sptr))

    def step():
        launch_fast()
        if world > 1:
            torch.distributed.all_gather_into_tensor(full.view(-1), y32.view(-1))

    L.check(L.lib.invop_apply(h, x32.data_ptr(), N, y32.data_ptr(), rows, k, L.F32, L.MODE_FAST,
                              C.c_void_p(sptr)), "apply")
    # operator bytes one apply streams (the layout the first apply built)
    op_bytes = C.c_int64()
    L.check(L.lib.invop_plan_apply_bytes(h, k, L.MODE_FAST, C.byref(op_bytes), C.c_void_p(sptr)))
    op_bytes = op_bytes.value
    # an operator shard that fits twice into L2 would be served from L2 in a
    # back-to-back loop: then every timed step gets its own event pair and a
    # write of 2x L2 between steps (outside the events)
    flush_l2 = op_bytes < 2 * L2_BYTES
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev) if flush_l2 else None
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()

    def timed(fn, reps):
        """Device milliseconds of `reps` calls of fn (CUDA events on the launching stream)."""
        if not flush_l2:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                fn()
            e1.record(stream)
            torch.cuda.synchronize()
            return e0.elapsed_time(e1)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
               for _ in range(reps)]
        for i in range(reps):
            flush.fill_(i)
            evs[i][0].record(stream)
            fn()
            evs[i][1].record(stream)
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in evs)

    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        lc0 = L.lib.invop_launch_count()
        ms = timed(step, args.steps)
        launches = L.lib.invop_launch_count() - lc0
    if world > 1:
        torch.distributed.barrier()
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps

    # ---- kernel-only timing of the apply launch(es) (dominant kernel) for the roofline
    kreps = max(20, min(args.steps, 2000 if k == 1 else 50))
    k_ms = timed(launch_fast, kreps) / kreps

    # ---- ordered (bitwise fp64) kernel for reference
    y64 = torch.empty((k, rows), dtype=torch.float64, device=dev)
    for _ in range(2):
        L.lib.invop_apply(h, x64.data_ptr(), N, y64.data_ptr(), rows, k, L.F64, L.MODE_ORDERED,
                          C.c_void_p(sptr))
    o0 = torch.cuda.Event(enable_timing=True)
    o1 = torch.cuda.Event(enable_timing=True)
    oreps = max(5, min(args.steps, 500 if k == 1 else 5))
    o0.record(stream)
    for _ in range(oreps):
        L.lib.invop_apply(h, x64.data_ptr(), N, y64.data_ptr(), rows, k, L.F64, L.MODE_ORDERED,
                          C.c_void_p(sptr))
    o1.record(stream)
    torch.cuda.synchronize()
    ord_ms = o0.elapsed_time(o1) / oreps

    # ---- end to end through the C ABI with host buffers (H2D + apply + D2H)
    xh = torch.from_numpy(np.ascontiguousarray(X)).pin_memory()
    yh = torch.empty((k, rows), dtype=torch.float64).pin_memory()
    for _ in range(2):
        L.check(L.lib.invop_apply_host(h, xh.data_ptr(), yh.data_ptr(), k, L.MODE_FAST,
                                       C.c_void_p(sptr)))
    e2e_steps = max(10, min(args.steps, 1000 if k == 1 else 30))
    if world > 1:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        L.lib.invop_apply_host(h, xh.data_ptr(), yh.data_ptr(), k, L.MODE_FAST, C.c_void_p(sptr))
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())

    # ---- correctness spot check of this run (fp32 path vs fp64 ordered, same codes)
    err = float(((y32.double() - y64).abs().max() / y64.abs().max()).item())
    # ---- quantization error: against the unquantized fp64 rows
    # of L^-1 (device block LU) applied to the same fp32-rounded x; Eq. 6 norm
    qerr = 0.0
    xr = x32.double()
    for b0 in range(0, rows, 4096):
        nb = min(4096, rows - b0)
        exact = dop.inverse_rows(row0 + b0, nb) @ xr.t()          # [nb, k]
        num = (y32[:, b0:b0 + nb].double().t() - exact).abs().amax(dim=0)
        if b0 == 0:
            qnum, qden = num, exact.abs().amax(dim=0)
        else:
            qnum = torch.maximum(qnum, num)
            qden = torch.maximum(qden, exact.abs().amax(dim=0))
        del exact
    if world > 1:
        torch.distributed.all_reduce(qnum, op=torch.distributed.ReduceOp.MAX)
        torch.distributed.all_reduce(qden, op=torch.distributed.ReduceOp.MAX)
    qerr = float((qnum / qden).max().item())
    del dop

    # ---- roofline of the dominant kernel (K2 fast, one launch per step)
    peak, peak_src = _peaks()
    code_bytes = plan.code_bytes
    kname = L.lib.invop_apply_kernel(h, k, L.MODE_FAST).decode()
    alg_bytes = op_bytes + k * N * 4 + k * rows * 4
    achieved = alg_bytes / (k_ms * 1e-3) / 1e9
    int8_ops = 2.0 * rows * N * k * (code_bytes * 3) if k > 1 else None
    traffic = None
    prof = ROOT / "profiles" / ("ncu_cfg%d_%s.json" % (cfg.key, kname))
    # the committed capture is of the whole operator on one GPU: it describes
    # a launch only when this rank holds all rows
    if prof.exists() and world == 1 and (not args.nrhs or args.nrhs == cfg.nrhs):
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:  # noqa: BLE001
            traffic = None

    result = None
    if rank == 0:
        mults, adds = plan.counts() if (world == 1 and N <= 16384) else (None, plan.counts()[1])
        value = k * args.steps / (ms * 1e-3)
        result = {
            "metric": METRIC,
            "value": value,
            "unit": UNIT,
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "strong",
            "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (seeded; BASELINE.json config %d; operator pinned in DESIGN.md)" % cfg.key,
            "config": {
                "workload": cfg.name, "N": N, "digits": cfg.digits, "nrhs": k,
                "rows_per_gpu": rows, "code_bytes_per_entry": code_bytes,
                "operator_bytes_per_gpu": op_bytes,
                "operator_bytes_per_entry": op_bytes / (rows * N),
                "parallelism": "row-shard x%d + all-gather" % world if world > 1 else "single GPU",
                "l2": ("operator shard %.0f MB < 2x L2: %d MB written between timed steps "
                       "(per-step CUDA events)" % (op_bytes / 1e6, 2 * L2_BYTES // 2**20))
                      if flush_l2 else
                      "inputs larger than L2 (operator %.0f MB streamed per apply vs 126 MB L2); no flush"
                      % (op_bytes / 1e6),
            },
            "roofline": {
                "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "%s (P=%d, %.3f operator B/entry)" % (kname, code_bytes, op_bytes / (rows * N)),
                "kernel_ms": k_ms,
                "algorithmic_bytes_per_launch": alg_bytes, "peak_source": peak_src,
            },
            "e2e": {
                "value": k * e2e_steps / e2e_s, "unit": UNIT,
                "h2d_bytes_per_step": k * N * 8, "d2h_bytes_per_step": k * rows * 8,
                "path": "invop_apply_host (C ABI, pinned host fp64 buffers)",
            },
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "ordered_fp64": {"value": k * 1e3 / ord_ms, "unit": UNIT, "kernel_ms": ord_ms,
                             "achieved_gbs": alg_bytes / (ord_ms * 1e-3) / 1e9,
                             "note": "bitwise equal to the reference apply"},
            "fp32_vs_fp64_relerr": err,
            "quantization_error": {"value": qerr, "digits": cfg.digits,
                                   "vs": "unquantized fp64 rows of L^-1 (device block LU), same x; "
                                         "max_i |y - y_exact| / max_i |y_exact|, worst RHS"},
            "setup_s": {"factor": t_factor, "construct_and_encode": t_setup - t_factor},
            "op_counters": {"multiplications": mults, "additions": adds},
        }
        if int8_ops:
            result["tensor"] = {"int8_ops_per_launch": int8_ops,
                                "achieved_tops": int8_ops / (k_ms * 1e-3) / 1e12,
                                "nominal_peak_tops": 4500.0,
                                "frac_of_nominal": int8_ops / (k_ms * 1e-3) / 1e12 / 4500.0,
                                "note": "dense int8 tensor peak not measured on this pool; nominal B200 figure"}
        if world == 1 and not args.no_cpu_baseline:
            result["cpu_baseline"] = cpu_baseline(cfg, budget_s=args.cpu_budget)
    return result


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nrhs", type=int, default=0,
                    help="right-hand sides per step (default: the config's own count)")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    args = ap.parse_args()
    world, rank, local = dist_init(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        res = run_ours(args, world, rank, local)
        if rank == 0 and res is not None:
            print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
