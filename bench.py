"""bench.py -- the driver's benchmark contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--n 8192] [--no-kernels] [--no-cpu] [--no-tune] [--e2e-steps E]

Headline workload (BASELINE.json configs[1]): FP32 matrix multiplication
n = 8192, program parameters auto-tuned inside the case the live B200
selects, rows of c sharded over the ranks (strong scaling: n is fixed).
A "step" is one pass of the hot path: one pk_launch of the selected leaf
over the resident inputs (c += a*b).  ``value`` is whole-job GFLOP/s from
CUDA events (max over ranks); ``e2e`` is the same metric through the C-ABI
host-buffer entry point pk_run_host with pinned host buffers (H2D of every
input and D2H of c inside the timed region).  The other BASELINE configs
(reversal, transpose, 1-D/2-D Jacobi, mat-vec) are measured in the same run
under ``kernels`` on rank 0 at N=1.

``--impl reference`` times the reference path's CPU restatement (the
oracle port, oracle/pk_oracle.c, all host threads) on a bounded sample of
the same workload -- the reference itself is a pure-Python interpreter
with no compiled form.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

MEASURED_PEAKS = os.path.join(REPO, "MEASURED_PEAKS.json")
NCU_TRAFFIC = os.path.join(REPO, "profiles", "ncu_traffic.json")
# which committed ncu capture describes each measured kernel (tools/make_profiles.py)
TRAFFIC_KEYS = {"matmul": "matmul_n8192", "reverse": "reverse_2p30", "transpose": "transpose_32768",
                "jacobi": "jacobi1d_2p28", "jacobi2d": "jacobi2d_16384", "matvec": "matvec_32768",
                "matvec_f32": "matvec_f32_32768", "addition": "addition_16384", "matmul_n2048": "matmul_n2048"}


def matmul_traffic_key(n: int, tuned: dict):
    """The committed capture of the FP32 matmul leaf the tuner picked: the
    128 x 128 tile (two CTAs per SM, or one with a producer warp when the tiles
    fill one wave) or the 128 x 64 tile; None for other tiles."""
    bn = tuned["ub1"] * tuned["s"]
    if tuned["B0"] != 128 or bn not in (64, 128) or n not in (2048, 8192):
        return None
    return "matmul_n%d" % n + ("" if bn == 128 else "_t64")


def traffic_entry(key: str, algorithmic: float):
    """The committed ncu capture's DRAM bytes per launch beside the algorithmic bytes."""
    rec = ncu_traffic(TRAFFIC_KEYS.get(key, key))
    if rec is None:
        return None
    return {"dram_bytes": rec["bytes"], "algorithmic_bytes": algorithmic, "ratio": round(rec["bytes"] / algorithmic, 4),
            "kernel": rec["kernel"], "source": rec["report"]}


def ncu_traffic(key: str):
    """DRAM bytes (read + write) per launch of the kernel captured under
    ``key`` by one ``ncu --set full`` run (profiles/ncu_traffic.json), or None."""
    try:
        with open(NCU_TRAFFIC) as fh:
            rec = json.load(fh).get(key)
    except (OSError, ValueError):
        return None
    return None if rec is None else {"bytes": rec["dram_bytes"], "kernel": rec["kernel"].split("(")[0],
                                     "report": "profiles/%s_ncu.md (%s)" % (rec["round"], rec["report"])}


FALLBACK_HBM_GBS = 6650.0  # B200_PROFILING.md fallback, used only without MEASURED_PEAKS.json
METRIC = "matmul GFLOP/s & stencil/reversal HBM GB/s, case-selected kernels, 1/2/4/8 B200"

# BASELINE.json configs measured under "kernels" (family, params, algorithmic bytes or flops)
KERNEL_CONFIGS = {
    "reverse": ({"N": 1 << 30, "s": 16, "B": 256}, 8 * (1 << 30), "GB/s"),
    "transpose": ({"N": 32768, "s": 8, "B0": 64, "B1": 8}, 8 * 32768 * 32768, "GB/s"),
    "jacobi": ({"T": 100, "N": (1 << 28) + 2, "s": 16, "B": 256}, 100 * 8 * (1 << 28), "GB/s"),
    "jacobi2d": ({"T": 50, "N": 16386, "s": 4, "B0": 8, "B1": 32}, 50 * 8 * 16384 * 16384, "GB/s"),
    "matvec": ({"N": 32768, "s": 1, "B": 128}, 4 * 32768 * 32768 + 8 * 32768, "GB/s"),
}


def load_peaks() -> dict:
    try:
        with open(MEASURED_PEAKS) as fh:
            d = json.load(fh)
        return {"hbm_gbs": float(d["hbm_gbs"]), "sm_max_mhz": float(d.get("sm_max_mhz", 1965.0)),
                "bf16_tflops": float(d.get("bf16_tflops", 2250.0)), "source": "measured (MEASURED_PEAKS.json)"}
    except (OSError, KeyError, ValueError):
        return {"hbm_gbs": FALLBACK_HBM_GBS, "sm_max_mhz": 1965.0, "bf16_tflops": 2250.0,
                "source": "fallback (B200_PROFILING.md)"}


# ----------------------------------------------------------------- clocks ----

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.FIELDS,
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
        return False

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in getattr(self, "lines", []):
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for name, val in zip(names, parts[3:7]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# --------------------------------------------------------------- helpers ----

def dist_info():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def cpu_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def timed_cpu(fn, budget_s: float, min_runs: int = 1):
    runs, t0 = 0, time.perf_counter()
    while True:
        fn()
        runs += 1
        el = time.perf_counter() - t0
        if runs >= min_runs and el >= budget_s:
            return el / runs, runs
        if el > budget_s * 3:
            return el / runs, runs


# ------------------------------------------------------------- reference ----

REF_ROWS = 64  # rows of the n = 8192 product per CPU step (8.6 GFLOP, ~0.1-0.2 s on 16 threads)


def reference_interp_rate(fam: str):
    """The reference interpreter's own rate (parakern.interp.run_program, one
    core), measured in the build container by tools/time_reference_interp.py:
    the reference cannot run on the GPU box."""
    try:
        with open(os.path.join(REPO, "profiles", "r02_reference_interp.json")) as fh:
            doc = json.load(fh)
    except (OSError, ValueError):
        return None
    rec = doc["families"].get(fam)
    if rec is None:
        return None
    return {"value": rec["value"], "unit": rec["unit"], "cores": 1, "points_per_s": rec["points_per_s"],
            "params": rec["params"], "where": doc["where"], "source": "profiles/r02_reference_interp.json"}


def run_reference(args) -> int:
    """The reference path on the host: the oracle port of interp.run_program
    (binary64, all host threads) on the headline's own workload -- FP32
    inputs of the n = 8192 matmul, each step a bounded block of REF_ROWS rows
    of the product -- so value and unit compare with our arm directly."""
    rank, world, _ = dist_info()
    if rank != 0:
        return 0
    import numpy as np

    from oracle import oracle

    n = args.n
    threads = cpu_cores()
    oracle.build()
    oracle.set_threads(threads)
    rng = np.random.default_rng(0x1801)
    a = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    b = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    c = np.zeros((n, n))
    P = {"n": n, "B0": 128, "ub1": 8, "s": 16}
    secs = []
    for i in range(args.warmup + args.steps):
        r0 = (i * REF_ROWS) % n
        t0 = time.perf_counter()
        oracle.matmul_rows_f64(P, r0, r0 + REF_ROWS, a, b, c)
        if i >= args.warmup:
            secs.append(time.perf_counter() - t0)
    sec = statistics.median(secs)
    gf = 2.0 * REF_ROWS * n * n / sec / 1e9
    sample = ("binary64 matmul of the n=%d workload (ascending k, unfused, the interpreter's order), "
              "rows [r0, r0+%d) per step (%.3g FLOP)" % (n, REF_ROWS, 2.0 * REF_ROWS * n * n))
    line = {
        "metric": METRIC, "impl": "reference", "value": round(gf, 3), "unit": "GFLOP/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 3),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic U[-1,1) fp32 inputs, seed 0x1801",
        "config": {"workload": "matmul n=%d fp32 FFMA, (B0,ub1,s) auto-tuned inside the live case" % n,
                   "n": n, "parallelism": "host threads", "sample_rows_per_step": REF_ROWS},
        "cpu_baseline": {"value": round(gf, 3), "unit": "GFLOP/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": round(gf, 3), "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_interpreter": reference_interp_rate("matmul"),
    }
    print(json.dumps(line), flush=True)
    return 0


def summary(line: dict) -> dict:
    """Compact per-family record at the end of the line: value, fraction of
    its roofline, the CPU port's rate on the box, and the parity verdict."""
    def verdict(p):
        if not p:
            return None
        return "ok" if (p.startswith("exact") or p.startswith("within")) else "FAIL"

    out = {"cols": ["value", "unit", "frac_roofline", "cpu_port", "parity"],
           "matmul_n%d" % line["config"]["n"]: [line["value"], "GFLOP/s", line["roofline"]["frac"],
                                                (line.get("cpu_baseline") or {}).get("value"),
                                                verdict(line.get("parity"))]}
    for fam, rec in (line.get("kernels") or {}).items():
        if not isinstance(rec, dict) or "value" not in rec or "temporal" in fam:
            continue
        frac = rec.get("frac_of_measured_hbm", rec.get("frac_of_fp32_peak", rec.get("frac_of_measured_hbm_x_n")))
        out[fam] = [rec["value"], rec["unit"], frac, (rec.get("cpu_baseline") or {}).get("value"),
                    verdict(rec.get("parity"))]
    if line.get("e2e"):
        out["e2e_c_abi"] = [line["e2e"]["value"], "GFLOP/s", None, None, None]
    if line.get("e2e_run_program"):
        out["e2e_run_program"] = [line["e2e_run_program"]["value"], "GFLOP/s", None, None, None]
    return out


# ------------------------------------------------------------------- ours ----

def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=8192)
    ap.add_argument("--no-kernels", action="store_true", help="skip the per-family extras")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-tune", action="store_true",
                    help="skip the tuners and use each grid's first entry (the recorded picks); "
                         "for profiler runs, whose timings are distorted")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_1801_04348_b200 import _lib, autotune, binding, cases, programs
    from paper_1801_04348_b200 import machine as machine_mod

    rank, world, local = dist_info()
    if world != args.gpus and world > 1:
        print("warning: WORLD_SIZE=%d but --gpus %d" % (world, args.gpus), file=sys.stderr)
    # test hook: PK_BENCH_ONE_GPU=1 maps every rank onto device 0 over gloo (the N > 1 code
    # path on a one-GPU box; NCCL refuses two ranks on one device)
    one_gpu = os.environ.get("PK_BENCH_ONE_GPU") == "1"
    if one_gpu:
        local = 0
    torch.cuda.set_device(local)
    if world > 1:
        if one_gpu:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        # one collective now, so the communicator exists (and is logged) before any timing
        probe = torch.ones(1, device=torch.device("cuda", local))
        dist.all_reduce(probe)
        print("bench: rank %d of %d on cuda:%d, backend %s, communicator ranks %d (all_reduce check %d)"
              % (rank, world, local, dist.get_backend(), dist.get_world_size(), int(probe.item())),
              file=sys.stderr, flush=True)
    dev = torch.device("cuda", local)
    peaks = load_peaks()
    mv = machine_mod.live(local)

    n = args.n
    kind = programs.original("matmul")
    base = {"n": n, "B0": 128, "ub1": 8, "s": 16}
    g = torch.Generator(device=dev)
    # one matmul over all ranks: the same a and b everywhere (the placement
    # partition.run_rows makes once, outside the timed region: b broadcast,
    # a/c rows scattered); each rank computes its rows of c, no collective
    g.manual_seed(0x1801)
    rows = n // world
    r0 = rank * rows
    a = torch.rand(n * n, device=dev, generator=g) * 2 - 1  # full-size buffers, rank owns its rows
    b = torch.rand(n * n, device=dev, generator=g) * 2 - 1
    c = torch.zeros(n * n, device=dev)
    ptrs = [a.data_ptr(), b.data_ptr(), c.data_ptr()]

    # tune (B0, ub1, s) inside the selected case, on this rank's shard
    grid = [{"B0": B0, "ub1": ub1, "s": s} for B0, ub1, s in
            ((128, 8, 8), (128, 8, 16), (64, 8, 16), (64, 8, 8), (64, 16, 8))]
    if args.no_tune:  # profiler runs: timings under ncu are distorted, use the recorded pick
        tuned, trials = dict(base, **grid[0]), []
    else:
        tuned, trials = autotune.autotune(kind, base, machine=mv, buffers=[a, b, c], reps=2, grid=grid)
    sel = cases.select(kind, tuned, mv)
    L = binding.make_launch(kind, tuned, sel.applied, _lib.DTYPE_F32, lo=r0, hi=r0 + rows)
    stream = torch.cuda.current_stream(dev)
    st = stream.cuda_stream

    for _ in range(max(3, args.warmup)):
        _lib.launch(L, ptrs, st)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            _lib.launch(L, ptrs, st)
        e1.record(stream)
        torch.cuda.synchronize()
    launches = _lib.launch_count() - launches0
    ms_local = e0.elapsed_time(e1)
    ms_t = torch.tensor([ms_local], device=dev)
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms_total = float(ms_t.item())
    ms_step = ms_total / args.steps
    flop_step = 2.0 * n * n * n  # whole job, all ranks
    value = flop_step / (ms_step * 1e-3) / 1e9

    # parity of the measured leaf at full size, outside the timed region: one
    # launch on fresh rows of c against a binary64 product of this rank's rows
    # (N > 1: every rank checks its own share, the worst error is reported)
    c.zero_()
    err_t = torch.tensor([matmul_error(L, [a, b, c], n, r0, r0 + rows)], device=dev)
    if world > 1:
        dist.all_reduce(err_t, op=dist.ReduceOp.MAX)
    headline_parity = parity_text(float(err_t.item()), n)

    # roofline of the dominant (only) kernel: FP32 FFMA pipe
    per_launch_flop = 2.0 * rows * n * n
    achieved_tf = per_launch_flop / (ms_local / args.steps * 1e-3) / 1e12
    sm_count = mv.props.get("sm_count", 148)
    peak_tf = sm_count * 256 * peaks["sm_max_mhz"] * 1e6 / 1e12
    clocks = clk.summary()
    peak_at_clock = sm_count * 256 * clocks["sm_mhz"] * 1e6 / 1e12 if clocks["sm_mhz"] else None

    # DRAM traffic of the dominant kernel per launch, from the committed ncu
    # capture of this exact configuration (one rank, the TMA-fed tile the tuner picked)
    headline_traffic = None
    tkey = matmul_traffic_key(n, tuned) if world == 1 else None
    if tkey:
        rec = ncu_traffic(tkey)
        headline_traffic = rec["bytes"] if rec else None

    # e2e through the C-ABI host-buffer call (pinned host memory)
    e2e = None
    ha = torch.empty(n * n, dtype=torch.float32, pin_memory=True)
    hb = torch.empty(n * n, dtype=torch.float32, pin_memory=True)
    hc = torch.zeros(n * n, dtype=torch.float32, pin_memory=True)
    ha.copy_(a.cpu())
    hb.copy_(b.cpu())
    Lh = binding.make_launch(kind, tuned, sel.applied, _lib.DTYPE_F32, lo=r0, hi=r0 + rows)
    hp = [ha.data_ptr(), hb.data_ptr(), hc.data_ptr()]
    for _ in range(max(3, args.warmup)):  # the allocator/stream pool and the first DMA of fresh pinned pages
        _lib.run_host(Lh, hp, local)
    if world > 1:
        dist.barrier()
    step_ms = []
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        t1 = time.perf_counter()
        _lib.run_host(Lh, hp, local)
        step_ms.append((time.perf_counter() - t1) * 1e3)
    e2e_s = torch.tensor([(time.perf_counter() - t0) / args.e2e_steps], device=dev)
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_gf = flop_step / float(e2e_s.item()) / 1e9
    # per rank: its rows of a and c in, all of b in, its rows of c out (pk_run_host copies the share)
    e2e = {"value": round(e2e_gf, 1), "unit": "GFLOP/s",
           "h2d_bytes_per_step": (2 * rows * n + n * n) * 4 * world,
           "d2h_bytes_per_step": rows * n * 4 * world,
           "ms_per_step_min_max": [round(min(step_ms), 3), round(max(step_ms), 3)],
           "path": "pk_run_host (C ABI) with pinned host buffers, rank share of a/c and all of b"}

    # the same call through the drop-in Python API with numpy host arrays
    # (run_program stages them into pooled pinned buffers and calls pk_run_host)
    e2e_api = None
    if world == 1:
        import numpy as np

        from paper_1801_04348_b200 import run_program

        na, nb = ha.numpy().reshape(n, n).copy(), hb.numpy().reshape(n, n).copy()
        nc = np.zeros((n, n), dtype=np.float32)
        text = programs.source("matmul")
        # warm-up as the timed loop runs: the staging ring, the pinned download
        # buffer and the result pool (a caller holding one result while the next
        # call runs keeps two result sets in the pool)
        out = None
        for _ in range(4):
            out = run_program(text, tuned, {"a": na, "b": nb, "c": nc})
        api_ms = []
        for _ in range(max(3, args.e2e_steps // 2)):
            t1 = time.perf_counter()
            out = run_program(text, tuned, {"a": na, "b": nb, "c": nc})
            api_ms.append((time.perf_counter() - t1) * 1e3)
        del out
        e2e_api = {"value": round(flop_step / (statistics.mean(api_ms) * 1e-3) / 1e9, 1), "unit": "GFLOP/s",
                   "h2d_bytes_per_step": 3 * n * n * 4, "d2h_bytes_per_step": n * n * 4,
                   "ms_per_step_min_max": [round(min(api_ms), 3), round(max(api_ms), 3)],
                   "path": "run_program(matmul.mfk, tuned, numpy float32 a/b/c in ordinary pageable memory): case "
                           "selection, pk_run_host_io reading the caller's arrays in place (staged through a pinned "
                           "ring inside the pipeline), a and b copied in the same pass, c into recycled host memory"}

    # optional 3xTF32 tcgen05 variant on the same shard (reported separately, never the headline)
    variants = {}
    try:
        Lt = binding.make_launch(kind, tuned, sel.applied, _lib.DTYPE_F32, lo=r0, hi=r0 + rows,
                                 extra_flags=_lib.FLAG_TF32X3)
        _lib.launch(Lt, ptrs, st)
        torch.cuda.synchronize()
        t0e, t1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0e.record(stream)
        for _ in range(args.steps):
            _lib.launch(Lt, ptrs, st)
        t1e.record(stream)
        torch.cuda.synchronize()
        ms_t = torch.tensor([t0e.elapsed_time(t1e) / args.steps], device=dev)
        if world > 1:
            dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        tf = flop_step / (float(ms_t.item()) * 1e-3) / 1e12
        variants["matmul_tf32x3_tcgen05"] = {
            "value": round(tf * 1e3, 1), "unit": "GFLOP/s (useful 2n^3)", "ms_per_step": round(float(ms_t.item()), 4),
            "tensor_tflops": round(3 * tf, 1),
            # dense TF32 is half the BF16 rate on B200 (1.1 vs 2.25 PFLOP/s nominal): the
            # measured BF16 burst / 2 is the measured-TF32 ceiling; the nominal one beside it
            # (per GPU: the value is the whole job's, over `world` GPUs)
            "frac_of_tf32_dense": round(3 * tf / world / (peaks.get("bf16_tflops", 2250.0) / 2), 4),
            "frac_of_tf32_nominal": round(3 * tf / world / (sm_count * 4096 * peaks["sm_max_mhz"] * 1e-6), 4),
            "note": "3xTF32 split (hi*hi + hi*lo + lo*hi) on tcgen05 kind::tf32, fp32 TMEM accumulation; "
                    "within the FP32 tolerance, not the FFMA path's rounding sequence"}
    except (NotImplementedError, ValueError, RuntimeError) as exc:  # shapes the variant does not tile
        variants["matmul_tf32x3_tcgen05"] = {"unavailable": str(exc)[:200]}

    kernels = {}
    cpu = None
    if world > 1 and not args.no_kernels:
        del ha, hb, hc
        kernels = bench_kernels_sharded(peaks, mv, rank, world)
    if rank == 0 and world == 1 and not args.no_kernels:
        del ha, hb, hc
        kernels = bench_kernels(peaks, mv, args.no_tune, cpu=not args.no_cpu)
        try:
            kernels["emitted_baseline"] = bench_emitted(kernels)
        except Exception as exc:  # the baseline is informative only
            kernels["emitted_baseline"] = {"unavailable": str(exc)[:200]}
    if rank == 0 and world == 1 and not args.no_cpu:
        # the same n = 8192 workload on the host: a row block of the product
        cpu = cpu_matmul_rows(n, 0, REF_ROWS, cpu_cores())
        cpu["reference_interpreter"] = reference_interp_rate("matmul")

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 1), "unit": "GFLOP/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic U[-1,1) fp32, seed 0x1801 (one matrix pair, rows of c sharded)",
            "config": {"workload": "matmul n=%d fp32 FFMA, (B0,ub1,s) auto-tuned inside the live case" % n,
                       "n": n, "tuned": tuned, "case": sel.index, "applied": list(sel.applied),
                       "machine": mv.values, "parallelism": "row-shard x%d" % world,
                       "l2": "inputs (3 x %d MiB) larger than L2" % (n * n * 4 >> 20),
                       "trials": [[t.params["B0"], t.params["ub1"], t.params["s"], round(t.ms, 3)] for t in trials]},
            "roofline": {"bound": "fp32-fma", "achieved": round(achieved_tf, 2),
                         "peak": round(peak_tf, 2), "unit": "TFLOP/s", "frac": round(achieved_tf / peak_tf, 4),
                         "peak_source": "computed: %d SM x 256 FLOP/clk x %.0f MHz max clock "
                                        "(MEASURED_PEAKS.json has no FP32 figure)" % (sm_count, peaks["sm_max_mhz"]),
                         "frac_at_observed_clock": round(achieved_tf / peak_at_clock, 4) if peak_at_clock else None,
                         "traffic": headline_traffic},
            "clocks": clocks,
            "e2e": e2e,
            "e2e_run_program": e2e_api,
            "parity": headline_parity,
            "gpu_launches": int(launches),
            "kernels": kernels,
            "variants": variants,
        }
        if cpu is not None:
            line["cpu_baseline"] = cpu
        line["summary"] = summary(line)  # last: the driver keeps the tail of stdout
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _fill(fam: str, shapes: dict, gen) -> list:
    """Synthetic int32 inputs of a family in declaration order.  Ranges keep
    every result inside int32 (mat-vec: |a|, |x| <= 2^7 at N = 32768), so the
    C-int kernels and the reference's unbounded ints agree exactly."""
    import torch

    from paper_1801_04348_b200 import programs

    lim = 1 << 7 if fam == "matvec" else 1 << 20
    bufs = []
    for arr in programs.FAMILIES[fam].arrays:
        n = 1
        for d in shapes[arr.name]:
            n *= d
        bufs.append(torch.randint(-lim, lim, (n,), dtype=torch.int32, device="cuda", generator=gen))
    return bufs


def restate(fam: str, P: dict, bufs: list) -> list:
    """What the program leaves in its arrays, restated with torch on the GPU
    from the initial contents (the checker of the bench's parity field; the
    same restatements as tests/test_gpu_parity.py)."""
    import torch

    out = [b.clone() for b in bufs]
    if fam == "reverse":
        N, tile = P["N"], P["s"] * P["B"]
        Pc = (N // tile) * tile
        out[1][N - Pc:] = torch.flip(bufs[0][:Pc], [0])
    elif fam == "transpose":
        N, I, J = P["N"], (P["N"] // P["B0"]) * P["B0"], (P["N"] // (P["s"] * P["B1"])) * P["s"] * P["B1"]
        out[1].view(N, N)[:I, :J] = bufs[0].view(N, N).t()[:I, :J]
    elif fam == "jacobi":
        N, tile = P["N"], P["s"] * P["B"]
        Pc = ((N - 2) // tile) * tile
        h = [out[0][:N], out[0][N:]]
        for t in range(P["T"]):
            src, dst = (h[1], h[0]) if t % 2 == 0 else (h[0], h[1])
            s = src[0:Pc].long() + src[1:Pc + 1] + src[2:Pc + 2]
            dst[1:Pc + 1] = torch.div(s, 3, rounding_mode="trunc").int()
    elif fam == "jacobi2d":
        N = P["N"]
        I, J = ((N - 2) // P["B0"]) * P["B0"], ((N - 2) // (P["s"] * P["B1"])) * P["s"] * P["B1"]
        a = out[0].view(2 * N, N)
        h = [a[:N], a[N:]]
        for t in range(P["T"]):
            src, dst = (h[0], h[1]) if t % 2 == 0 else (h[1], h[0])
            s = (src[0:I, 1:J + 1].long() + src[2:I + 2, 1:J + 1] + src[1:I + 1, 0:J] + src[1:I + 1, 2:J + 2]
                 + src[1:I + 1, 1:J + 1])
            dst[1:I + 1, 1:J + 1] = torch.div(s, 5, rounding_mode="trunc").int()
    elif fam == "matvec":
        N, tile = P["N"], P["s"] * P["B"]
        R = (N // tile) * tile
        a = bufs[0].view(N, N)[:R].double()
        out[2][:R] = (bufs[2][:R].double() + a @ bufs[1].double()).round().int()  # |sums| < 2^53: exact
    elif fam == "addition":
        N = P["N"]
        I = (N // P["B0"]) * P["B0"]
        J, half = min((N // (2 * P["B1"])) * P["B1"], N // 2), N // 2
        a, b, c = (x.view(N, N) for x in (bufs[0], bufs[1], out[2]))
        c[:I, :J] = a[:I, :J] + b[:I, :J]
        c[:I, half:half + J] = a[:I, half:half + J] + b[:I, half:half + J]
    else:
        raise KeyError(fam)
    return out


def parity_check(fam: str, P: dict, L, gen) -> str:
    """One run of the measured leaf on fresh inputs, outside the timed
    region, against restate(): "exact" or the first mismatch."""
    import torch

    from paper_1801_04348_b200 import _lib, programs

    bufs = _fill(fam, programs.array_shapes(programs.original(fam), P), gen)
    want = restate(fam, P, bufs)
    _lib.launch(L, [b.data_ptr() for b in bufs], torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    for i, (g, w) in enumerate(zip(bufs, want)):
        if not torch.equal(g, w):
            bad = int((g != w).nonzero()[0, 0])
            return "MISMATCH array %d at %d" % (i, bad)
    return "exact"


# bounded CPU samples of each family for the oracle port (all host threads)
CPU_SAMPLES = {
    "reverse": ({"N": 1 << 27, "s": 16, "B": 256}, lambda P: 8 * P["N"], "GB/s"),
    "transpose": ({"N": 8192, "s": 8, "B0": 64, "B1": 8}, lambda P: 8 * P["N"] ** 2, "GB/s"),
    "jacobi": ({"T": 4, "N": (1 << 26) + 2, "s": 16, "B": 256}, lambda P: P["T"] * 8 * (P["N"] - 2), "GB/s"),
    "jacobi2d": ({"T": 4, "N": 4098, "s": 4, "B0": 8, "B1": 32}, lambda P: P["T"] * 8 * (P["N"] - 2) ** 2, "GB/s"),
    "matvec": ({"N": 16384, "s": 1, "B": 512}, lambda P: 4 * P["N"] ** 2 + 8 * P["N"], "GB/s"),
    "addition": ({"N": 8192, "B0": 8, "B1": 128}, lambda P: 12 * P["N"] ** 2, "GB/s"),
}


def cpu_sample(fam: str, threads: int) -> dict:
    """The reference path's CPU restatement (oracle/pk_oracle.c, OpenMP over
    all host threads) on a bounded sample of the family's workload."""
    import numpy as np

    from oracle import oracle
    from paper_1801_04348_b200 import programs

    oracle.build()
    oracle.set_threads(threads)
    P, work, unit = CPU_SAMPLES[fam]
    shapes = programs.array_shapes(programs.original(fam), P)
    rng = np.random.default_rng(0x1801)
    lim = 1 << 7 if fam == "matvec" else 1 << 20
    arrays = {k: rng.integers(-lim, lim, size=v, dtype=np.int32) for k, v in shapes.items()}
    oracle.run(fam, dict(P, T=1) if "T" in P else P, arrays)  # page in, warm the threads
    sec, runs = timed_cpu(lambda: oracle.run(fam, P, arrays), budget_s=1.0)
    return {"value": round(work(P) / sec / 1e9, 3), "unit": unit, "cores": threads, "kind": "port",
            "sample": "oracle/pk_oracle.c on %s, %.3f s/run x %d" % (json.dumps(P), sec, runs)}


def bench_kernels(peaks, mv, no_tune: bool = False, cpu: bool = True) -> dict:
    """The bandwidth-bound BASELINE configs on one GPU: GB/s of algorithmic
    traffic and the fraction of the measured copy bandwidth, each with a
    parity check of the measured leaf at full size and the oracle port's
    rate on a bounded CPU sample."""
    import torch

    from paper_1801_04348_b200 import _lib, autotune, binding, cases, programs

    out = {}
    threads = cpu_cores()
    gen = torch.Generator(device="cuda")
    for fam, (params, work, unit) in KERNEL_CONFIGS.items():
        kind = programs.original(fam)
        shapes = programs.array_shapes(kind, params)
        gen.manual_seed(0x1801)
        bufs = _fill(fam, shapes, gen)
        ptrs = [x.data_ptr() for x in bufs]
        # tune (B, s) / (B0, B1, s) inside the live case on 4 time steps, run the full T
        # (2 steps x 2 launches picked a 6 % slower 1-D leaf on one box: too short to time)
        tune_base = dict(params, T=4) if "T" in params else dict(params)
        if no_tune:
            tuned, trials = dict(tune_base, **TUNE_GRIDS[fam][0]), []
        else:
            tuned, trials = autotune.autotune(kind, tune_base, machine=mv, buffers=bufs,
                                              reps=4 if "T" in params else 2, grid=TUNE_GRIDS.get(fam))
        run_params = dict(tuned, T=params["T"]) if "T" in params else tuned
        sel = cases.select(kind, run_params, mv)
        L = binding.make_launch(kind, run_params, sel.applied, _lib.DTYPE_I32)
        st = torch.cuda.current_stream()
        _lib.launch(L, ptrs, st.cuda_stream)
        torch.cuda.synchronize()
        reps = 1 if fam.startswith("jacobi") else 5
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(reps):
            _lib.launch(L, ptrs, st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = work / (ms * 1e-3) / 1e9
        out[fam] = {"params": run_params, "case": sel.index, "applied": list(sel.applied), "ms": round(ms, 3),
                    "value": round(gbs, 1), "unit": unit, "frac_of_measured_hbm": round(gbs / peaks["hbm_gbs"], 4),
                    "frac_of_8tbs": round(gbs / 8000.0, 4), "tuning_trials": len(trials)}
        rec = ncu_traffic(TRAFFIC_KEYS[fam])
        if rec and run_params == dict(params, **TUNE_GRIDS[fam][0]):
            # per launch (per sweep for the stencils) from the committed ncu capture
            per = (work / params["T"]) if "T" in params else work
            out[fam]["traffic"] = {"dram_bytes": rec["bytes"], "algorithmic_bytes": per,
                                   "ratio": round(rec["bytes"] / per, 4), "kernel": rec["kernel"],
                                   "source": rec["report"]}
        if fam in ("jacobi", "jacobi2d"):  # temporally blocked variant, reported separately (same results)
            for h in ((7, 15) if fam == "jacobi" else (3, 7)):
                Lt = binding.make_launch(kind, run_params, sel.applied, _lib.DTYPE_I32,
                                         extra_flags=_lib.FLAG_TEMPORAL)
                Lt.tblock = h
                _lib.launch(Lt, ptrs, st.cuda_stream)
                torch.cuda.synchronize()
                e0.record(st)
                _lib.launch(Lt, ptrs, st.cuda_stream)
                e1.record(st)
                torch.cuda.synchronize()
                tms = e0.elapsed_time(e1)
                tg = work / (tms * 1e-3) / 1e9
                out["%s_temporal_h%d" % (fam, h)] = {
                    "params": run_params, "ms": round(tms, 3), "value": round(tg, 1), "unit": unit,
                    "speedup_vs_per_step": round(ms / tms, 2),
                    "note": "algorithmic bytes of the per-step program / time: exceeds the HBM roofline "
                            "because h steps share one HBM pass; results bit-identical"}
        del bufs
        torch.cuda.empty_cache()
        out[fam]["parity"] = parity_check(fam, run_params, L, gen)
        torch.cuda.empty_cache()
        if cpu:
            try:
                out[fam]["cpu_baseline"] = cpu_sample(fam, threads)
            except Exception as exc:  # informative only
                out[fam]["cpu_baseline"] = {"unavailable": str(exc)[:200]}
    # mat-vec on float32 data (SURVEY 8(d) proposes N = 32768 FP32): double-float accumulation
    if "matvec" in out and "params" in out["matvec"]:
        mp = dict(out["matvec"]["params"])
        Nm = mp["N"]
        kind = programs.original("matvec")
        sel = cases.select(kind, mp, mv)
        L = binding.make_launch(kind, mp, sel.applied, _lib.DTYPE_F32)
        g = torch.Generator(device="cuda").manual_seed(0x1801)
        bufs = [torch.rand(Nm * Nm, device="cuda", generator=g) * 2 - 1, torch.rand(Nm, device="cuda", generator=g),
                torch.zeros(Nm, device="cuda")]
        ptrs = [x.data_ptr() for x in bufs]
        st = torch.cuda.current_stream()
        for _ in range(3):
            _lib.launch(L, ptrs, st.cuda_stream)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(10):
            _lib.launch(L, ptrs, st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        gbs = (4 * Nm * Nm + 8 * Nm) / (ms * 1e-3) / 1e9
        # parity: one launch from y = 0 against a binary64 product, 2 fp32 ulps
        bufs[2].zero_()
        _lib.launch(L, ptrs, st.cuda_stream)
        want = bufs[0].view(Nm, Nm).double() @ bufs[1].double()
        ok = bool(((bufs[2].double() - want).abs() <= 2 * 2.0**-24 * want.abs() + 1e-30).all())
        out["matvec_f32"] = {"params": mp, "case": sel.index, "applied": list(sel.applied), "ms": round(ms, 3),
                             "value": round(gbs, 1), "unit": "GB/s",
                             "frac_of_measured_hbm": round(gbs / peaks["hbm_gbs"], 4),
                             "parity": "within 2 fp32 ulps of binary64" if ok else "MISMATCH",
                             "traffic": traffic_entry("matvec_f32", 4 * Nm * Nm + 8 * Nm),
                             "note": "float32 a, x, y; products split exactly and summed as a double-float pair"}
        del bufs, want
        torch.cuda.empty_cache()
        if cpu:
            out["matvec_f32"]["cpu_baseline"] = cpu_matvec_f32(threads)
    out["matmul_n1024_table"] = bench_matmul_table(peaks, mv, threads if cpu else 0, no_tune)
    out["addition"] = bench_addition(peaks, mv, threads if cpu else 0)
    out["matmul_n2048"] = bench_matmul_n2048(peaks, mv, no_tune, threads if cpu else 0)
    return out


# the paper's Table of matmul thread blocks (ub1, B0) x s
PAPER_SHAPES = [(16, 4), (32, 4), (64, 4), (8, 8), (16, 8), (32, 8), (64, 8)]


def bench_matmul_table(peaks, mv, threads: int, no_tune: bool = False) -> dict:
    """BASELINE configs[0]: FP32 matmul n = 1024 with the case discussion
    evaluated for the reference's default machine model (fermi.machine) at
    the paper's Table shapes; each selected leaf runs on the B200 with the
    program's own thread mapping (the generic kernel: a B0 x ub1 block per
    B0 x ub1*s tile), beside the leaf the live machine tunes."""
    import torch

    from paper_1801_04348_b200 import _lib, binding, cases, programs

    n = 1024
    kind = programs.original("matmul")
    g = torch.Generator(device="cuda").manual_seed(0x1801)
    bufs = [torch.rand(n * n, device="cuda", generator=g) * 2 - 1 for _ in range(3)]
    ptrs = [x.data_ptr() for x in bufs]
    st = torch.cuda.current_stream()
    peak = mv.props.get("sm_count", 148) * 256 * peaks["sm_max_mhz"] * 1e6 / 1e9
    rows, worst = [], 0.0
    for ub1, B0 in PAPER_SHAPES:
        for s in (2, 4):
            P = {"n": n, "B0": B0, "ub1": ub1, "s": s}
            sel = cases.select(kind, P, "fermi")
            L = binding.make_launch(kind, P, sel.applied, _lib.DTYPE_F32)
            _lib.launch(L, ptrs, st.cuda_stream)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record(st)
            for _ in range(5):
                _lib.launch(L, ptrs, st.cuda_stream)
            e1.record(st)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            bufs[2].zero_()
            worst = max(worst, matmul_error(L, bufs, n, 0, n))
            rows.append([ub1, B0, s, sel.index, list(sel.applied), round(2.0 * n ** 3 / (ms * 1e-3) / 1e9, 1)])
    best = max(r[5] for r in rows)
    # (B0, ub1, s) tuned inside the case the live machine selects (coverage-preserving candidates)
    from paper_1801_04348_b200 import autotune

    grid = [{"B0": B0, "ub1": ub1, "s": s} for B0, ub1, s in ((64, 8, 8), (128, 8, 16), (64, 8, 16), (128, 8, 8))]
    base = {"n": n, "B0": 64, "ub1": 8, "s": 8}
    if no_tune:
        P, trials = dict(base), []
    else:
        P, trials = autotune.autotune(kind, base, machine=mv, buffers=bufs, reps=20, grid=grid)
    L = binding.make_launch(kind, P, cases.select(kind, P, mv).applied, _lib.DTYPE_F32)
    for _ in range(3):
        _lib.launch(L, ptrs, st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(50):  # ~50 us launches: a longer window than the 17 ms headline's 10
        _lib.launch(L, ptrs, st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    tuned = 2.0 * n ** 3 / (e0.elapsed_time(e1) / 50 * 1e-3) / 1e9
    bufs[2].zero_()
    worst = max(worst, matmul_error(L, bufs, n, 0, n))
    del bufs
    torch.cuda.empty_cache()
    rec = {"value": round(tuned, 1), "unit": "GFLOP/s", "frac_of_fp32_peak": round(tuned / peak, 4),
           "tuned_params": P, "paper_shapes": {"cols": ["ub1", "B0", "s", "fermi case", "applied", "GFLOP/s"],
                                               "rows": rows, "best": best},
           "parity": parity_text(worst, n),
           "tuning_trials": len(trials),
           "note": "every Table shape selects fermi case 1 (no strategies) at n = 1024, as the survey found; "
                   "value = the leaf tuned inside the live B200's case; the Table shapes run the program's own "
                   "thread mapping"}
    if threads:
        rec["cpu_baseline"] = cpu_matmul_rows(n, 0, n, threads)
    return rec


def bench_addition(peaks, mv, threads: int) -> dict:
    """addition.mfk, N = 16384: 12 bytes per element."""
    import torch

    from paper_1801_04348_b200 import _lib, binding, cases, programs

    P = {"N": 16384, "B0": 8, "B1": 128}
    kind = programs.original("addition")
    sel = cases.select(kind, P, mv)
    L = binding.make_launch(kind, P, sel.applied, _lib.DTYPE_I32)
    gen = torch.Generator(device="cuda").manual_seed(0x1801)
    bufs = _fill("addition", programs.array_shapes(kind, P), gen)
    ptrs = [x.data_ptr() for x in bufs]
    st = torch.cuda.current_stream()
    for _ in range(3):
        _lib.launch(L, ptrs, st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(10):
        _lib.launch(L, ptrs, st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    work = 12 * P["N"] ** 2
    gbs = work / (ms * 1e-3) / 1e9
    del bufs
    torch.cuda.empty_cache()
    rec = {"params": P, "case": sel.index, "applied": list(sel.applied), "ms": round(ms, 3), "value": round(gbs, 1),
           "unit": "GB/s", "frac_of_measured_hbm": round(gbs / peaks["hbm_gbs"], 4),
           "parity": parity_check("addition", P, L, gen), "traffic": traffic_entry("addition", work)}
    if threads:
        rec["cpu_baseline"] = cpu_sample("addition", threads)
    return rec


def bench_matmul_n2048(peaks, mv, no_tune: bool, threads: int) -> dict:
    """The other size of BASELINE configs[1]: FP32 matmul n = 2048, (B0, ub1, s)
    tuned inside the case."""
    import torch

    from paper_1801_04348_b200 import _lib, autotune, binding, cases, programs

    n2 = 2048
    kind = programs.original("matmul")
    base = {"n": n2, "B0": 128, "ub1": 8, "s": 16}
    g = torch.Generator(device="cuda").manual_seed(0x1801)
    bufs = [torch.rand(n2 * n2, device="cuda", generator=g) * 2 - 1 for _ in range(3)]
    grid = [{"B0": B0, "ub1": ub1, "s": s} for B0, ub1, s in ((128, 8, 16), (128, 8, 8), (64, 8, 16), (64, 8, 8))]
    if no_tune:
        tuned, trials = dict(base), []
    else:
        # the candidates are within 1-3 % of each other here: time them over as
        # many launches as the measurement below (5 launches misranked them)
        tuned, trials = autotune.autotune(kind, base, machine=mv, buffers=bufs, reps=20, grid=grid)
    sel = cases.select(kind, tuned, mv)
    L = binding.make_launch(kind, tuned, sel.applied, _lib.DTYPE_F32)
    ptrs = [x.data_ptr() for x in bufs]
    st = torch.cuda.current_stream()
    for _ in range(3):
        _lib.launch(L, ptrs, st.cuda_stream)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(50):  # ~0.28 ms launches: a 14 ms window
        _lib.launch(L, ptrs, st.cuda_stream)
    e1.record(st)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 50
    gf = 2.0 * n2 ** 3 / (ms * 1e-3) / 1e9
    peak = mv.props.get("sm_count", 148) * 256 * peaks["sm_max_mhz"] * 1e6 / 1e9
    bufs[2].zero_()
    err = matmul_error(L, bufs, n2, 0, n2)
    rec = {"params": tuned, "case": sel.index, "applied": list(sel.applied), "ms": round(ms, 4),
           "value": round(gf, 1), "unit": "GFLOP/s", "frac_of_fp32_peak": round(gf / peak, 4),
           "tuning_trials": len(trials), "parity": parity_text(err, n2),
           "traffic": traffic_entry(matmul_traffic_key(n2, tuned), 4.0 * n2 * n2 * 4)
           if matmul_traffic_key(n2, tuned) else None}
    del bufs
    torch.cuda.empty_cache()
    if threads:
        rec["cpu_baseline"] = cpu_matmul_rows(n2, 0, n2, threads)
    return rec


def matmul_error(L, bufs, n: int, r0: int, r1: int) -> float:
    """One launch of L on (a, b, c) and the normalised error of rows [r0, r1)
    of c against a binary64 product: max|C - C64| / max sum_k |a_ik b_kj|."""
    import torch

    from paper_1801_04348_b200 import _lib

    a, b, c = (x.view(n, n) for x in bufs)
    c0 = c[r0:r1].double()
    _lib.launch(L, [x.data_ptr() for x in bufs], torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    a64, b64 = a[r0:r1].double(), b.double()
    want = c0 + a64 @ b64
    scale = (a64.abs() @ b64.abs()).max()
    return float(((c[r0:r1].double() - want).abs().max() / scale).item())


def parity_text(err: float, K: int) -> str:
    tol = max(1e-5 * K / 1024.0, 2.0 * K * 2.0**-24)
    return "%s: normalised error %.3g vs tolerance %.3g (1e-5*K/1024)" % ("within" if err <= tol else "MISMATCH",
                                                                         err, tol)


def cpu_matvec_f32(threads: int) -> dict:
    """float32 mat-vec by the oracle port (binary64 sums, all host threads) on
    an N = 16384 sample of the N = 32768 workload, GB/s of a-traffic."""
    import numpy as np

    from oracle import oracle

    oracle.build()
    oracle.set_threads(threads)
    N = 16384
    rng = np.random.default_rng(0x1801)
    arrays = {"a": rng.uniform(-1, 1, (N, N)).astype(np.float32), "x": rng.uniform(-1, 1, N).astype(np.float32)}
    P = {"N": N, "s": 1, "B": 512}
    oracle.run("matvec", P, arrays)
    sec, runs = timed_cpu(lambda: oracle.run("matvec", P, arrays), budget_s=1.0)
    return {"value": round((4 * N * N + 8 * N) / sec / 1e9, 3), "unit": "GB/s", "cores": threads, "kind": "port",
            "sample": "oracle/pk_oracle.c float32 mat-vec (binary64 sums) N=%d, %.3f s/run x %d" % (N, sec, runs)}


def cpu_matmul_rows(n: int, r0: int, r1: int, threads: int) -> dict:
    """Rows [r0, r1) of the n x n matmul in binary64 by the oracle port (all
    host threads): a bounded sample of the same workload, GFLOP/s."""
    import numpy as np

    from oracle import oracle

    oracle.build()
    oracle.set_threads(threads)
    rng = np.random.default_rng(0x1801)
    a = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    b = rng.uniform(-1, 1, (n, n)).astype(np.float32)
    c = np.zeros((n, n))
    P = {"n": n, "B0": 128, "ub1": 8, "s": 16}
    oracle.matmul_rows_f64(P, r0, min(r1, r0 + 8), a, b, c)  # warm the threads
    sec, runs = timed_cpu(lambda: oracle.matmul_rows_f64(P, r0, r1, a, b, c), budget_s=1.0)
    flop = 2.0 * (r1 - r0) * n * n
    return {"value": round(flop / sec / 1e9, 3), "unit": "GFLOP/s", "cores": threads, "kind": "port",
            "sample": "oracle/pk_oracle.c binary64 matmul n=%d, rows [%d, %d) of the product (%.3g FLOP), "
                      "%.3f s/run x %d" % (n, r0, r1, flop, sec, runs)}


def _owned_slices(fam: str, P: dict, lo: int, hi: int) -> list:
    """(array index, start, end) of the flat elements units [lo, hi) write --
    a rank's share of the result."""
    from paper_1801_04348_b200 import partition, programs

    if hi <= lo:
        return []
    if fam == "jacobi":
        N = P["N"]
        return [(0, lo, hi), (0, N + lo, N + hi)]
    if fam == "jacobi2d":
        N = P["N"]
        return [(0, lo * N, hi * N), (0, (N + lo) * N, (N + hi) * N)]
    names = [a.name for a in programs.FAMILIES[fam].arrays]
    out = []
    for w in programs.FAMILIES[fam].written:
        off, cnt = partition.share_range(fam, P, w, lo, hi)
        out.append((names.index(w), off, off + cnt))
    return out


def bench_kernels_sharded(peaks, mv, rank: int, world: int) -> dict:
    """The bandwidth-bound BASELINE configs over all ranks (N > 1), placed by
    the partitioner: reversal by input element, transpose / mat-vec by output
    row (no data-path collective), the stencils by row slab with ghost zones
    of width h refreshed every h steps by NCCL send/recv over NVLink
    (partition.run_stencil).  GB/s of whole-job algorithmic traffic over the
    max-over-ranks device time; the leaf parameters are each family's
    recorded tuner pick (TUNE_GRIDS[fam][0])."""
    import torch
    import torch.distributed as dist

    from paper_1801_04348_b200 import _lib, binding, cases, partition, programs

    out = {}
    dev = torch.device("cuda", torch.cuda.current_device())
    st = torch.cuda.current_stream(dev)
    for fam, (params, work, unit) in KERNEL_CONFIGS.items():
        try:
            kind = programs.original(fam)
            run_params = dict(params, **TUNE_GRIDS[fam][0])
            sel = cases.select(kind, run_params, mv)
            shapes = programs.array_shapes(kind, run_params)
            g = torch.Generator(device=dev)
            g.manual_seed(0x1801)  # the same inputs on every rank
            bufs = []
            for arr in programs.FAMILIES[fam].arrays:
                n = 1
                for d in shapes[arr.name]:
                    n *= d
                bufs.append(torch.randint(-(1 << 20), 1 << 20, (n,), dtype=torch.int32, device=dev, generator=g))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            if fam in ("jacobi", "jacobi2d"):
                L = binding.make_launch(kind, dict(run_params, T=1), sel.applied, _lib.DTYPE_I32)
                if _lib.jacobi_narrow(L, bufs[0].data_ptr(), st.cuda_stream):
                    L.flags |= _lib.FLAG_NARROW
                ex = partition.TorchExchanger()
                plan = partition.halo_plan(fam, run_params, rank, world, width=16)

                def sweep(src, dst, lo, hi, L=L):
                    _lib.jacobi_sweep(L, src.data_ptr(), dst.data_ptr(), lo, hi, st.cuda_stream)

                def run():
                    partition.drive(partition.run_stencil(fam, run_params, bufs[0], ex, sweep, plan=plan))
                detail = {"ghost_width": plan.width, "slab": [plan.lo, plan.hi]}
            else:
                lo, hi = partition.unit_range_launch(fam, run_params, rank, world)
                L = binding.make_launch(kind, run_params, sel.applied, _lib.DTYPE_I32, lo=lo, hi=hi)
                ptrs = [x.data_ptr() for x in bufs]

                def run(L=L, ptrs=ptrs, lo=lo, hi=hi):
                    if hi > lo:
                        for _ in range(5):
                            _lib.launch(L, ptrs, st.cuda_stream)
                detail = {"units": [lo, hi]}
            run()  # warm-up
            torch.cuda.synchronize()
            dist.barrier()
            e0.record(st)
            run()
            e1.record(st)
            torch.cuda.synchronize()
            reps = 1 if fam.startswith("jacobi") else 5
            ms = torch.tensor([e0.elapsed_time(e1) / reps], device=dev)
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            ms = float(ms.item())
            gbs = work / (ms * 1e-3) / 1e9
            out[fam] = {"params": run_params, "case": sel.index, "applied": list(sel.applied), "ms": round(ms, 3),
                        "value": round(gbs, 1), "unit": unit, "n_gpus": world,
                        "frac_of_measured_hbm_x_n": round(gbs / (peaks["hbm_gbs"] * world), 4),
                        "placement": detail if rank == 0 else None}
            # parity of this rank's share at full size (outside the timed region):
            # fresh inputs, one run, the written share against restate()
            g.manual_seed(0x1801)
            fresh = _fill(fam, shapes, g)
            want = restate(fam, run_params, fresh)
            for b, f in zip(bufs, fresh):
                b.copy_(f)
            del fresh
            if fam in ("jacobi", "jacobi2d"):
                run()
                owned = _owned_slices(fam, run_params, plan.lo, plan.hi)
            else:
                if hi > lo:
                    _lib.launch(L, ptrs, st.cuda_stream)
                owned = _owned_slices(fam, run_params, lo, hi)
            torch.cuda.synchronize()
            ok = all(torch.equal(bufs[i][o0:o1], want[i][o0:o1]) for i, o0, o1 in owned)
            ok_t = torch.tensor([0 if ok else 1], device=dev)
            dist.all_reduce(ok_t, op=dist.ReduceOp.MAX)
            out[fam]["parity"] = "exact (every rank's share)" if int(ok_t.item()) == 0 else "MISMATCH"
            del want
            if fam in ("jacobi", "jacobi2d"):
                # the same slabs with the halo exchange fused into the sweep: ghost units
                # stored straight into the neighbours' buffers over NVLink (CUDA IPC), no NCCL
                g.manual_seed(0x1801)
                bufs[0].copy_(torch.randint(-(1 << 20), 1 << 20, bufs[0].shape, dtype=torch.int32, device=dev,
                                            generator=g))
                ps = partition.PeerStencil(fam, run_params, bufs[0], L)
                ps.run(params["T"])  # warm-up
                ps.finish()
                ps.ctr.zero_()
                g.manual_seed(0x1801)  # the timed run starts from fresh inputs (checked below)
                bufs[0].copy_(_fill(fam, shapes, g)[0])
                torch.cuda.synchronize()
                dist.barrier()
                e0.record(st)
                for t in range(params["T"]):
                    _lib.jacobi_sweep_peer(L, bufs[0].data_ptr(), t, ps.lo, ps.hi, ps.peer, st.cuda_stream)
                e1.record(st)
                torch.cuda.synchronize()
                # the timed run started from the fresh inputs: check this rank's slab
                g.manual_seed(0x1801)
                init = _fill(fam, shapes, g)
                want = restate(fam, run_params, init)
                del init
                ps_ok = all(torch.equal(bufs[0][o0:o1], want[0][o0:o1])
                            for _, o0, o1 in _owned_slices(fam, run_params, ps.lo, ps.hi))
                del want
                ok_t = torch.tensor([0 if ps_ok else 1], device=dev)
                dist.all_reduce(ok_t, op=dist.ReduceOp.MAX)
                ps.close()
                pms = torch.tensor([e0.elapsed_time(e1)], device=dev)
                dist.all_reduce(pms, op=dist.ReduceOp.MAX)
                pms = float(pms.item())
                pg = work / (pms * 1e-3) / 1e9
                out[fam + "_peer"] = {"params": run_params, "ms": round(pms, 3), "value": round(pg, 1), "unit": unit,
                                      "n_gpus": world, "frac_of_measured_hbm_x_n": round(pg / (peaks["hbm_gbs"] * world), 4),
                                      "parity": "exact (every rank's slab)" if int(ok_t.item()) == 0 else "MISMATCH",
                                      "exchange": "fused into the sweep: ghost units stored into the neighbours' "
                                                  "buffers through CUDA IPC (NVLink), device counters, no NCCL"}
            del bufs
            torch.cuda.empty_cache()
        except Exception as exc:  # informative extras: never lose the headline line
            out[fam] = {"unavailable": ("%s: %s" % (type(exc).__name__, exc))[:200]}
    return out


EMITTED_CONFIGS = {
    # program: (params, algorithmic work, unit) -- the reference's emitted leaf text
    # (static shared memory, grid capped at 256 blocks), compiled with NVRTC
    "reverse": ({"N": 1 << 30, "s": 16, "B": 256}, 8 * (1 << 30), "GB/s"),
    "transpose": ({"N": 32768, "s": 4, "B0": 32, "B1": 8}, 8 * 32768 * 32768, "GB/s"),
    "jacobi": ({"T": 10, "N": (1 << 28) + 2, "s": 16, "B": 256}, 10 * 8 * (1 << 28), "GB/s"),
    "matvec": ({"N": 8192, "s": 1, "B": 256}, 4 * 8192 * 8192 + 8 * 8192, "GB/s"),
    "matmul": ({"n": 4096, "B0": 32, "ub1": 8, "s": 4}, 2 * 4096**3, "GFLOP/s"),
}


def bench_emitted(ours: dict) -> dict:
    """The "naive emitted kernel" bar: the reference's own
    CUDA text for the original program, compiled for sm_100a at load time."""
    import torch

    from paper_1801_04348_b200 import jit

    path = os.path.join(REPO, "tests", "golden", "emitted_leaves.json")
    with open(path) as fh:
        entries = {(e["program"], e["variant"]): e for e in json.load(fh)["entries"]}
    out = {}
    for prog, (params, work, unit) in EMITTED_CONFIGS.items():
        leaf = jit.Leaf.from_json(entries[(prog, "original")]["leaf"])
        shapes = jit.array_shapes(leaf, params)
        bufs = {}
        for name, shape in shapes.items():
            n = jit.eval_product(shape)
            if unit == "GFLOP/s":
                bufs[name] = torch.randint(-4, 4, (n,), dtype=torch.int32, device="cuda")
            else:
                bufs[name] = torch.randint(-(1 << 20), 1 << 20, (n,), dtype=torch.int32, device="cuda")
        st = torch.cuda.current_stream()
        jit.run_leaf(leaf, params, bufs, st.cuda_stream)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        jit.run_leaf(leaf, params, bufs, st.cuda_stream)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        val = work / (ms * 1e-3) / 1e9
        out[prog] = {"params": params, "ms": round(ms, 3), "value": round(val, 1), "unit": unit,
                     "kernel": leaf.kernel_name}
        del bufs
        torch.cuda.empty_cache()
    return out


# candidate program parameters per family (warp-multiple blocks; coverage-preserving
# ones are kept by the tuner).  The first entry of each grid is the tuner's pick on
# B200 in the last measured run (profiles/r01*_bench.json), used by --no-tune.
TUNE_GRIDS = {
    "reverse": [{"B": b, "s": s} for b, s in ((256, 16), (128, 32), (512, 8), (1024, 4), (256, 8))],
    "transpose": [{"B0": b0, "B1": b1, "s": s} for b0, b1, s in ((64, 8, 8), (32, 8, 4), (64, 16, 4),
                                                                 (32, 32, 1), (128, 8, 4))],
    "jacobi": [{"B": b, "s": s} for b, s in ((256, 16), (256, 8), (128, 32), (512, 8), (1024, 4))],
    "jacobi2d": [{"B0": b0, "B1": b1, "s": s} for b0, b1, s in ((64, 4, 32), (8, 32, 16), (32, 8, 32),
                                                                (32, 8, 16), (16, 16, 32))],
    "matvec": [{"B": b, "s": s} for b, s in ((256, 1), (128, 1), (64, 2), (512, 1), (32, 4))],
}


if __name__ == "__main__":
    raise SystemExit(main())
