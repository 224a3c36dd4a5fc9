"""Benchmark: quantized inverse-operator applies/s and achieved HBM GB/s.

BASELINE.json metric: "inverse-operator applies/sec and achieved HBM GB/s
(frac of roofline) at N=128^2" — config 4 (variable-eps, non-uniform
128x128 grid, N=16384, 5 decimal digits, single fp32 right-hand side).

A step is one apply y = L_eps^-1 rho of the quantized operator resident in
HBM (one K2 launch; for N>1 plus the NCCL all-gather of the row shards and
the unshard kernel). The operator streamed per apply (424 MB at config 4) is
larger than 2x L2, so no L2 flush is needed between steps; shards that would
fit are flushed (config["l2"]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4]
    python bench.py --impl reference ...   # the reference's CPU kernel

Under torchrun each rank owns a contiguous row block of L^-1 (built on its
own GPU by the block-LU constructor), applies it to rho, and the row blocks
are all-gathered: the operator is fixed, so the scaling is strong and the
line reports whole-job applies/s. Rank 0 prints one JSON line.

--impl reference times the reference's own compiled plan_apply (oracle/_ref,
built from /root/reference's _native.pyx) on the host, over the whole
quantized operator when it fits the run (config 4 at the driver's step
counts), else on a column sample scaled by N/cols.
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
def _dist1() -> bool:
    """INVOP_BENCH_DIST1=1: run the N>1 code path (NCCL all-gather, unshard,
    graph capture) with a one-rank process group - the only way to exercise it
    on a one-GPU box."""
    return bool(os.environ.get("INVOP_BENCH_DIST1"))


def dist_init(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 or (_dist1() and args.impl == "ours"):
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        os.environ.setdefault("RANK", "0")
        os.environ.setdefault("WORLD_SIZE", "1")
        import torch
        import torch.distributed as dist

        backend = "nccl" if args.impl == "ours" else "gloo"
        if backend == "nccl":
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
    return world, rank, local


# ------------------------------------------------------------------ workload
def workload_config(cfg, world: int, k: int) -> dict:
    """The `config` object of the JSON line: a function of the workload and
    N only, so both arms (ours, --impl reference) print the same one."""
    from paper_1602_00001_b200.sharded import shard_rows

    N = cfg.N
    rows = shard_rows(N, world, 0)[1]          # the largest shard
    # every device layout stores >= 1 byte per entry: a shard below 2x L2
    # could be served from L2 in a back-to-back loop, so those runs flush
    flush = rows * N < 2 * L2_BYTES
    return {
        "workload": cfg.name, "N": N, "digits": cfg.digits, "nrhs": k,
        "rows_per_gpu": rows,
        "parallelism": "row-shard x%d + one all-gather" % world if world > 1 else "single GPU",
        "l2": ("operator shard < 2x L2: 256 MB written between timed steps (per-step events)"
               if flush else "operator shard larger than 2x L2 (126 MB); no flush"),
    }


def _rhs(cfg, nrhs: int) -> np.ndarray:
    X = cfg.rhs()
    if nrhs:
        reps = -(-nrhs // X.shape[0])
        X = np.ascontiguousarray(np.tile(X, (reps, 1))[:nrhs])
    return X


def _mem_available() -> int:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 0


# ------------------------------------------------------------------ reference (CPU)
def reference_full(cfg):
    """The whole quantized operator of `cfg` as the reference builds it —
    dense L^-1 by LU + solve on the identity (dense.py:36-62), quantize
    (quant.py:48-65), build_plan's CSC tables (applyplan.py:116-172, restated
    in C with threads: the numpy lexsort takes minutes at N=16384) — and the
    reference's own compiled plan_apply (oracle/_ref)."""
    from oracle import invop_oracle as O

    st = cfg.operator()
    t0 = time.perf_counter()
    inv = O.invert_dense(st.to_sparse().toarray())
    t1 = time.perf_counter()
    mant = O.quantize(inv, cfg.digits)
    del inv
    t2 = time.perf_counter()
    plan = O.build_plan_large(mant, cfg.digits)
    del mant
    t3 = time.perf_counter()
    return plan, {"invert": t1 - t0, "quantize": t2 - t1, "build_plan": t3 - t2}


def reference_sample(cfg, target_step_s: float = 0.25, seed_cols: int = 7):
    """Bounded sample of the workload for the reference CPU kernel: C columns
    of the quantized L^-1 (host sparse LU, reference rounding, reference
    grouping restated), all rows; a step's time is scaled by N/C."""
    from oracle import invop_oracle as O
    import scipy.sparse.linalg as spla

    st = cfg.operator()
    N = st.n
    rng = np.random.default_rng(seed_cols)
    lu = spla.splu(st.to_sparse().tocsc())

    def make(cols):
        J = np.sort(rng.choice(N, size=cols, replace=False))
        E = np.zeros((N, cols))
        E[J, np.arange(cols)] = 1.0
        mant = O.quantize(lu.solve(E), cfg.digits)       # columns J of L^-1
        return J, O.build_plan_rect(mant, cfg.digits)

    ref = O.reference_native()
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

    cols = 256
    J, plan = make(cols)
    scale = max(0.05, min(16.0, target_step_s / max(run(J, plan), 1e-6)))
    cols = int(min(N, max(16, cols * scale)))
    J, plan = make(cols)
    return dict(J=J, plan=plan, run=run, cols=cols, N=N,
                kind="reference" if ref is not None else "port")


def cpu_baseline(cfg, budget_s: float = 15.0):
    """`cpu_baseline` of our line: ~budget_s of reference plan_apply on a
    column sample of the workload (single-threaded: the reference holds the GIL)."""
    s = reference_sample(cfg)
    times = []
    t_end = time.perf_counter() + budget_s
    while time.perf_counter() < t_end or len(times) < 3:
        times.append(s["run"](s["J"], s["plan"]))
        if len(times) >= 50:
            break
    per_apply = min(times) * s["N"] / s["cols"]
    return {
        "value": 1.0 / per_apply,
        "unit": UNIT,
        "cores": 1,
        "kind": s["kind"],
        "sample": "%d of %d columns of the quantized L^-1 (all %d rows), reference plan_apply "
                  "best of %d runs, scaled by N/cols (extrapolated); single-threaded (the "
                  "reference holds the GIL)" % (s["cols"], s["N"], s["N"], len(times)),
        "host_cpus": os.cpu_count(),
        "affinity_cpus": len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else None,
    }


def run_reference(args, world, rank):
    """--impl reference: the reference's own compiled plan_apply
    (_native.pyx:15-49, built from its source into oracle/_ref) on the host
    cores, through its own table format, on our arm's workload. Never loads
    libinvop_b200.so (the package's library is dlopen'ed lazily)."""
    from paper_1602_00001_b200 import configs
    from oracle import invop_oracle as O

    if rank != 0:
        return
    cfg = configs.get(args.config)
    X = _rhs(cfg, args.nrhs)
    k, N = X.shape
    ref = O.reference_native()
    kind = "reference" if ref is not None else "port"
    line = {
        "impl": "reference", "metric": METRIC, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded; BASELINE.json config %d)" % cfg.key,
        "config": workload_config(cfg, world, k),
    }
    # whole-operator timing when it fits the host and the run stays short:
    # one step = k full applies (~2.5 ns per entry on one core)
    est_step = k * N * N * 2.5e-9
    need = 48 * N * N                          # dense fp64 inverse + LU + tables
    full = (ref is not None and N * N <= 2 ** 29 and _mem_available() > need
            and (args.steps + args.warmup) * est_step <= 240.0)
    if full:
        plan, setup = reference_full(cfg)
        args_t = (plan["col_ptr"], plan["group_coeff"], plan["group_ptr"], plan["entry_rows"],
                  plan["entry_signs"])

        def step():
            for t in range(k):
                ref.plan_apply(*args_t, X[t], np.zeros(N))

        for _ in range(args.warmup):
            step()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        el = time.perf_counter() - t0
        value = k * args.steps / el
        sample = ("whole operator: the reference's plan_apply over all %d x %d entries (%d groups, "
                  "%d entries) per RHS, every step" % (N, N, plan["group_ptr"].size - 1,
                                                       plan["entry_rows"].size))
        line["setup_s"] = setup
    else:
        target = max(0.005, min(0.2, 60.0 / max(1, args.steps + args.warmup)))
        s = reference_sample(cfg, target_step_s=target)
        for _ in range(args.warmup):
            s["run"](s["J"], s["plan"])
        t0 = time.perf_counter()
        for _ in range(args.steps):
            s["run"](s["J"], s["plan"])
        el = time.perf_counter() - t0
        value = 1.0 / (el / args.steps * s["N"] / s["cols"])
        sample = ("%d of %d columns per step, scaled by N/cols (extrapolated: the whole operator "
                  "does not fit this run's time or memory budget)" % (s["cols"], s["N"]))
    line.update({
        "value": value, "ms_per_step": k * 1e3 / value,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": 1, "kind": kind, "sample": sample,
                         "host_cpus": os.cpu_count()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })
    # the reference arm never touches this repo's native library
    from paper_1602_00001_b200 import _lib as _L

    line["b200_library_loaded"] = _L.loaded()
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ our arm
def _int8_peak():
    p = ROOT / "profiles" / "int8_tc_peak.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["tops"]), "measured (%s)" % p.relative_to(ROOT)
    return None, "unmeasured"


def quantization_error(cfg, X32: np.ndarray, Y: np.ndarray) -> float:
    """the apply against a direct sparse solve of the
    unquantized operator, y_exact = splu(A).solve(x) on the same fp32-rounded
    x; Eq. 6 normalisation (reference bench.py:73-85), worst RHS."""
    import scipy.sparse.linalg as spla

    A = cfg.operator().to_sparse().tocsc()
    lu = spla.splu(A)
    Xd = X32.astype(np.float64)
    exact = lu.solve(np.ascontiguousarray(Xd.T)).T          # [k, N]
    num = np.abs(Y - exact).max(axis=1)
    den = np.abs(exact).max(axis=1)
    return float((num / den).max())


def run_ours(args, world, rank, local):
    import ctypes as C

    import torch

    import paper_1602_00001_b200 as invop
    from paper_1602_00001_b200 import configs, _lib as L
    from paper_1602_00001_b200.sharded import row_offsets, shard_rows

    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    # the sharded step (apply + all-gather + unshard, graph capture, max over
    # ranks); INVOP_BENCH_DIST1 takes it with a one-rank group as well
    multi = world > 1 or _dist1()
    cfg = configs.get(args.config)
    st = cfg.operator()
    N = st.n
    row0, rows = shard_rows(N, world, rank)
    pad = shard_rows(N, world, 0)[1]
    offs = row_offsets(N, world)
    # ---- setup (timed separately): block-LU factor + construct + encode
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dop = invop.DeviceOperator(st).factor()
    torch.cuda.synchronize()
    t_factor = time.perf_counter() - t0
    plan = dop.quantized_rows(cfg.digits, row0, rows)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    del dop

    X = _rhs(cfg, args.nrhs)
    k = X.shape[0]
    x32 = torch.tensor(X, dtype=torch.float32, device=dev)      # [k, N], resident
    x64 = x32.double()
    stage = torch.empty((world, k, pad), dtype=torch.float32, device=dev)
    mine = stage[rank]
    # one right-hand side and an even row split: the gathered slices already
    # are y in row order, no reassembly launch
    y_is_stage = k == 1 and N % world == 0
    Y = stage.view(1, N) if y_is_stage else torch.empty((k, N), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    sptr = C.c_void_p(stream.cuda_stream)
    h = plan.handle

    def launch_fast():
        L.lib.invop_apply(h, x32.data_ptr(), N, mine.data_ptr(), pad, k, L.F32, L.MODE_FAST, sptr)

    def step_eager():
        # the stream is looked up per call: under graph capture it is the
        # capture stream
        sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        L.lib.invop_apply(h, x32.data_ptr(), N, mine.data_ptr(), pad, k, L.F32, L.MODE_FAST, sp)
        if multi:
            torch.distributed.all_gather_into_tensor(stage.view(-1), mine.reshape(-1))
            if not y_is_stage:
                L.lib.invop_unshard(stage.data_ptr(), world, offs.ctypes.data, k, pad, Y.data_ptr(), N,
                                    L.F32, sp)

    step = step_eager

    L.check(L.lib.invop_apply(h, x32.data_ptr(), N, mine.data_ptr(), pad, k, L.F32, L.MODE_FAST,
                              sptr), "apply")
    op_bytes = C.c_int64()
    L.check(L.lib.invop_plan_apply_bytes(h, k, L.MODE_FAST, C.byref(op_bytes), sptr))
    op_bytes = op_bytes.value
    ord_bytes = C.c_int64()
    L.check(L.lib.invop_plan_apply_bytes(h, k, L.MODE_ORDERED, C.byref(ord_bytes), sptr))
    ord_bytes = ord_bytes.value
    tc_ops = C.c_int64()
    L.check(L.lib.invop_plan_tensor_ops(h, k, L.MODE_FAST, C.byref(tc_ops), sptr))
    tc_ops = tc_ops.value
    flush_l2 = rows * N < 2 * L2_BYTES
    flush = torch.empty(2 * L2_BYTES // 4, dtype=torch.int32, device=dev) if flush_l2 else None
    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if multi:
        torch.distributed.barrier()
    # N > 1: a step is three launches and a collective issued from Python; at a
    # few GPUs the per-step host time exceeds the per-rank device time, so the
    # step is captured once in a CUDA graph (apply + all-gather + unshard) and
    # replayed. Kept eager if capture fails (the line says which). N = 1 stays
    # eager: consecutive k2_dl applies overlap as programmatic dependents.
    graph_used = False
    graph_launches = 0
    if (multi or os.environ.get("INVOP_BENCH_GRAPH")) and not os.environ.get("INVOP_BENCH_NO_GRAPH"):
        try:
            g = torch.cuda.CUDAGraph()
            cs = torch.cuda.Stream()
            cs.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(cs):
                step_eager()                       # warm the capture stream
            torch.cuda.current_stream().wait_stream(cs)
            torch.cuda.synchronize()
            lcg = L.lib.invop_launch_count()
            with torch.cuda.graph(g, stream=cs):
                step_eager()
            graph_launches = L.lib.invop_launch_count() - lcg      # library kernels per replay
            torch.cuda.synchronize()
            g.replay()
            torch.cuda.synchronize()
            step = g.replay
            graph_used = True
        except Exception as e:  # noqa: BLE001
            print("bench: CUDA graph capture failed, eager steps (%s)" % e, file=sys.stderr)
            torch.cuda.synchronize()
        if multi:
            ok = torch.tensor([1 if graph_used else 0], device=dev)
            torch.distributed.all_reduce(ok, op=torch.distributed.ReduceOp.MIN)
            if int(ok.item()) == 0:
                step, graph_used = step_eager, False    # every rank the same way
            torch.distributed.barrier()

    def timed(fn, reps, sync_each=False):
        """Device ms of `reps` calls of fn (CUDA events on the launching stream);
        per-call event pairs (+ L2 flush between calls when needed, or a host
        synchronisation after each call for the isolated-launch figure)."""
        if not flush_l2 and not sync_each:
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
            if flush_l2:
                flush.fill_(i)
            evs[i][0].record(stream)
            fn()
            evs[i][1].record(stream)
            if sync_each:
                torch.cuda.synchronize()
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in evs)

    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if multi:
            torch.distributed.barrier()
        lc0 = L.lib.invop_launch_count()
        ms = timed(step, args.steps)
        launches = L.lib.invop_launch_count() - lc0
        if graph_used:                    # replays do not pass through the library
            launches = graph_launches * args.steps
    if multi:
        torch.distributed.barrier()
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps

    # ---- the apply alone (dominant kernel(s)): back to back, and isolated
    kreps = max(20, min(args.steps, 2000 if k == 1 else 50))
    k_ms = timed(launch_fast, kreps) / kreps
    ireps = max(10, min(args.steps, 200 if k == 1 else 20))
    iso_ms = timed(launch_fast, ireps, sync_each=True) / ireps

    # ---- ordered (bitwise fp64) kernel
    y64 = torch.empty((k, rows), dtype=torch.float64, device=dev)

    def launch_ordered():
        L.lib.invop_apply(h, x64.data_ptr(), N, y64.data_ptr(), rows, k, L.F64, L.MODE_ORDERED, sptr)

    for _ in range(2):
        launch_ordered()
    oreps = max(5, min(args.steps, 500 if k == 1 else 5))
    ord_ms = timed(launch_ordered, oreps) / oreps

    # ---- end to end with host buffers
    if not multi:
        xh = torch.from_numpy(np.ascontiguousarray(X)).pin_memory()        # fp64 host
        yh = torch.empty((k, rows), dtype=torch.float64).pin_memory()

        def e2e_step():
            L.lib.invop_apply_host(h, xh.data_ptr(), yh.data_ptr(), k, L.MODE_FAST, sptr)

        e2e_h2d, e2e_d2h = k * N * 8, k * rows * 8
        e2e_path = "invop_apply_host (C ABI, pinned host fp64 x in, fp64 y out)"
    else:
        xh = torch.from_numpy(np.ascontiguousarray(X.astype(np.float32))).pin_memory()
        yh = torch.empty((k, N), dtype=torch.float32).pin_memory()

        def e2e_step():
            x32.copy_(xh, non_blocking=True)
            step()
            yh.copy_(Y, non_blocking=True)
            stream.synchronize()

        e2e_h2d, e2e_d2h = k * N * 4, k * N * 4
        e2e_path = "pinned fp32 x -> device, sharded apply + all-gather + unshard, full Y -> pinned host"
    for _ in range(2):
        e2e_step()
    e2e_steps = max(10, min(args.steps, 1000 if k == 1 else 30))
    if multi:
        torch.distributed.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        e2e_step()
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if multi:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        e2e_s = float(t.item())

    # ---- the drop-in default (bitwise fp64) end to end with host buffers
    ord_e2e = None
    if not multi and k == 1:
        yh64 = torch.empty((k, rows), dtype=torch.float64).pin_memory()

        def e2e_ordered():
            L.lib.invop_apply_host(h, xh.data_ptr(), yh64.data_ptr(), k, L.MODE_ORDERED, sptr)

        for _ in range(2):
            e2e_ordered()
        n_o = max(10, min(args.steps, 300))
        t0 = time.perf_counter()
        for _ in range(n_o):
            e2e_ordered()
        torch.cuda.synchronize()
        ord_e2e = k * n_o / (time.perf_counter() - t0)

    # ---- result of this run: full Y (gathered), fp32 vs the ordered fp64 path
    step()
    torch.cuda.synchronize()
    y32 = (Y if multi else mine[:, :rows]).double()
    y32_local = mine[:, :rows].double()
    err = float(((y32_local - y64).abs().amax(dim=1) / y64.abs().amax(dim=1)).max().item())
    Yh = y32.cpu().numpy()
    if multi:
        t = torch.tensor([err], dtype=torch.float64, device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        err = float(t.item())

    peak, peak_src = _peaks()
    kname = L.lib.invop_apply_kernel(h, k, L.MODE_FAST).decode()
    alg_bytes = op_bytes + k * N * 4 + k * rows * 4
    achieved = alg_bytes / (k_ms * 1e-3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / ("ncu_cfg%d_%s.json" % (cfg.key, kname))
    if prof.exists() and not multi and (not args.nrhs or args.nrhs == cfg.nrhs):
        try:
            traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
        except Exception:  # noqa: BLE001
            traffic = None

    result = None
    if rank == 0:
        mults, adds = plan.counts() if (not multi and N <= 16384) else (None, plan.counts()[1])
        value = k * args.steps / (ms * 1e-3)
        result = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded; BASELINE.json config %d; operator pinned in DESIGN.md)" % cfg.key,
            "config": workload_config(cfg, world, k),
            "layout": {
                "kernel": kname, "code_bytes_per_entry": plan.code_bytes,
                "operator_bytes_per_gpu": op_bytes,
                "operator_bytes_per_entry": op_bytes / (rows * N),
                "l2_flush_between_steps": flush_l2,
            },
            "roofline": {
                "bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "kernel": "%s (P=%d, %.3f operator B/entry)" % (kname, plan.code_bytes, op_bytes / (rows * N)),
                "kernel_ms": k_ms,
                "algorithmic_bytes_per_launch": alg_bytes, "peak_source": peak_src,
                "isolated": {"kernel_ms": iso_ms,
                             "achieved": alg_bytes / (iso_ms * 1e-3) / 1e9,
                             "frac": alg_bytes / (iso_ms * 1e-3) / 1e9 / peak,
                             "note": "one apply per host synchronisation (no overlap with a "
                                     "preceding apply)"},
            },
            "e2e": {"value": k * e2e_steps / e2e_s, "unit": UNIT,
                    "h2d_bytes_per_step": e2e_h2d, "d2h_bytes_per_step": e2e_d2h, "path": e2e_path},
            "gpu_launches": launches,
            "cuda_graph": graph_used,
            "clocks": clk.summary(),
            "ordered_fp64": {"value": k * 1e3 / ord_ms, "unit": UNIT, "kernel_ms": ord_ms,
                             "operator_bytes": ord_bytes,
                             "achieved_gbs": (ord_bytes + k * N * 8 + k * rows * 8) / (ord_ms * 1e-3) / 1e9,
                             "kernel": L.lib.invop_apply_kernel(h, k, L.MODE_ORDERED).decode(),
                             "e2e": ord_e2e,
                             "note": "bitwise equal to the reference apply; bytes = the byte planes "
                                     "it streams; e2e = invop_apply_host in ordered mode "
                                     "(pinned fp64 x in, fp64 y out, synchronous), applies/s"},
            "fp32_vs_fp64_relerr": err,
            "setup_s": {"factor": t_factor, "construct_and_encode": t_setup - t_factor},
            "op_counters": {"multiplications": mults, "additions": adds},
        }
        if tc_ops:
            tops = tc_ops / (k_ms * 1e-3) / 1e12
            pk, pk_src = _int8_peak()
            result["tensor"] = {"int8_ops_per_launch": tc_ops, "achieved_tops": tops,
                                "peak_tops": pk, "peak_source": pk_src,
                                "frac": tops / pk if pk else None,
                                "note": "2*M*N*K over the kind::i8 MMAs the kernel issues"}
        if not args.no_quant_error:
            result["quantization_error"] = {
                "value": quantization_error(cfg, X.astype(np.float32), Yh), "digits": cfg.digits,
                "vs": "direct sparse solve of the unquantized operator (scipy splu), same fp32 x; "
                      "max_i |y - y_exact| / max_i |y_exact|, worst RHS"}
        if not multi and not args.no_cpu_baseline:
            result["cpu_baseline"] = cpu_baseline(cfg, budget_s=args.cpu_budget)
    return result


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--nrhs", type=int, default=0,
                    help="right-hand sides per step (default: the config's own count)")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-quant-error", action="store_true")
    args = ap.parse_args()
    world, rank, local = dist_init(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
    else:
        res = run_ours(args, world, rank, local)
        if rank == 0 and res is not None:
            print(json.dumps(res), flush=True)
    if world > 1 or (_dist1() and args.impl == "ours"):
        import torch.distributed as dist

        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
