#!/usr/bin/env python
"""Throughput of the multi-amplitude XEB hot path on B200 (BASELINE.json).

Workload (BASELINE.json configs[1], "cfg2"): synthetic 30-qubit 5x6 grid,
m=12 (grid_circuit seed 12345, fused), 10^4 uniformly random bitstrings
(seed 99), the reference-annealed plan plans/cfg2.plan with 4 sliced legs
(16 slices). One step = every slice of the whole evaluation + the slice sum
(+ one NCCL reduce when N>1) + the fused |amp|^2 -> linear-XEB reduction.

    python bench.py [--gpus N] [--steps K] [--warmup W]           # this engine
    python bench.py --impl reference [...]                        # reference CPU

N>1 runs under torchrun: one process per GPU, slices split into contiguous
blocks, partial amplitudes summed by one NCCL reduce to rank 0.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("amplitudes/sec and effective TFLOP/s (complex64) for batched XEB at "
          "1/2/4/8 B200")
WORKLOADS = {
    "cfg1": dict(rows=3, cols=4, layers=8, k=1000,
                 text="cfg1: synthetic 12-qubit 3x4 grid, m=8 (grid_circuit seed 12345, "
                      "fused), 1000 random bitstrings (seed 99), plans/cfg1.plan (no slicing)"),
    "cal45": dict(rows=4, cols=5, layers=10, k=1000,
                  text="cal45: synthetic 20-qubit 4x5 grid, m=10 (grid_circuit seed 12345, fused), "
                       "1000 random bitstrings (seed 99), plans/cal45.plan (3 sliced legs); the "
                       "reference arm's calibration run"),
    "cfg3": dict(kind="sycamore", cycles=12, circuit_seed=2024, k=10000, row_chunk=10000, rows=0, cols=53,
                 text="cfg3: synthetic 53-qubit Sycamore layout, m=12 (ABCDCDAB fSim, sycamore_circuit seed "
                      "2024, fused), 10^4 random bitstrings (seed 99), plans/cfg3.plan (20 sliced legs, 2^20 "
                      "slices; plans/sycamore_plan.py), all requests' memo tables resident (84 GB arena)"),
    "cfg4": dict(kind="sycamore", cycles=14, circuit_seed=2024, k=100000, row_chunk=25000, rows=0, cols=53,
                 text="cfg4: synthetic 53-qubit Sycamore layout, m=14 (ABCDCDAB fSim, sycamore_circuit seed "
                      "2024, fused), 10^5 random bitstrings (seed 99), plans/cfg4.plan (24 sliced legs, 2^24 "
                      "slices; plans/sycamore_plan.py), memo streaming in chunks of 25,000 requests"),
    "cfg2": dict(rows=5, cols=6, layers=12, k=10000,
                 text="cfg2: synthetic 30-qubit 5x6 grid, m=12 (grid_circuit seed 12345, "
                      "fused), 10^4 random bitstrings (seed 99), plans/cfg2.plan "
                      "(4 sliced legs, 16 slices)"),
}


def load_workload(name: str, k: int = 0):
    from workloads import network as N
    from paper_2108_05665_b200.engine import problem_arrays

    w = WORKLOADS[name]
    if w.get("kind") == "sycamore":
        c = N.sycamore_circuit(w["cycles"], w["circuit_seed"])
        bits = N.random_bitstrings(N.Rng(99), c.n_qubits, w["k"])[: k or w["k"]]
        d = N.to_diagram(c, True)
        asg = N.build_assignments(d, bits, [])
        # MTCG_PLAN_FILE: a candidate plan instead of the committed one (plan search A/B)
        plan_text = open(os.environ.get("MTCG_PLAN_FILE") or os.path.join(ROOT, "plans", f"{name}.plan")).read()
        return problem_arrays(N.parse_plan(plan_text), d, asg), c, bits, plan_text
    c = N.grid_circuit(w["rows"], w["cols"], w["layers"], 12345)
    bits = N.random_bitstrings(N.Rng(99), w["rows"] * w["cols"], w["k"])
    d = N.to_diagram(c, True)
    asg = N.build_assignments(d, bits, [])
    plan_text = open(os.path.join(ROOT, "plans", f"{name}.plan")).read()
    plan = N.parse_plan(plan_text)
    return problem_arrays(plan, d, asg), c, bits, plan_text


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), float(p["bf16_tflops"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, 1590.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        self.first = ""
        if os.environ.get("BENCH_NO_CLOCKS"):
            self.proc = None
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            # wait for the first sample: nvidia-smi's start-up (NVML init) must
            # not overlap the timed region
            self.first = self.proc.stdout.readline()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def __exit__(self, *exc):
        self.out = ""
        if self.proc:
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) != 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# The one full run of the reference on the bench workload (cfg2): the
# unmodified reference's eval_sliced over all 16 slices with 8 workers in the
# dev container (8-core Xeon), tests/golden/make_cfg2_reference.py, which also
# wrote tests/golden/cfg2_reference.npz; the contract_pair sampler below
# estimated 1,667 s for that same run on that host.
CFG2_FULL_RUN = {"seconds": 3952.0, "threads": 8, "host": "dev container, 8-core Intel Xeon",
                 "sampler_estimate_seconds": 1667.0,
                 "source": "tests/golden/make_cfg2_reference.py (DESIGN.md §5b)"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ref_problem(R, name: str):
    """The workload built by the REFERENCE's own producers: its grid_circuit
    and random_bitstrings test generators (proj/tests/support/gen.cpp:54-107)
    and its circuit / diagram / assignment / plan parsers."""
    w = WORKLOADS[name]
    circ = R.grid_circuit(w["rows"], w["cols"], w["layers"], 12345)
    bits = R.random_bitstrings(99, w["rows"] * w["cols"], w["k"])
    plan = open(os.path.join(ROOT, "plans", f"{name}.plan")).read()
    return R.RefProblem(circ, bits, plan, fuse=True)


def ref_calibration(R, threads: int):
    """Real end-to-end runs of the unmodified reference on this host, timed
    beside the sampler's estimate of the same runs: cal45 (4x5 grid, m=10,
    10^3 bitstrings, 3 sliced legs; eval_sliced with all threads) and cfg1
    (eval_all, single-threaded by the reference's contract)."""
    out = {}
    for name, mode, workers in (("cal45", "sliced", threads), ("cfg1", "all", 1)):
        p = ref_problem(R, name)
        S = 1 << len(p.plan_sliced())
        p.eval(mode, workers)  # warm
        best = min(_timed(lambda: p.eval(mode, workers)) for _ in range(3))
        est1, _, _ = p.sample_eval_time(1 << 24, threads)
        est = est1 / min(workers, S)
        out[name] = {"real_seconds": best, "sampler_seconds": est, "ratio": best / est,
                     "workers": workers, "amplitudes_per_s": p.n_requests / best,
                     "mode": f"eval_{mode}"}
    return out


def _timed(f):
    t0 = time.perf_counter()
    f()
    return time.perf_counter() - t0


def cpu_baseline(threads: int, config: str = "cfg2"):
    """The reference CPU path on this host, on a bounded sample of the same
    workload, entirely through oracle/_ref (the unmodified reference library;
    nothing of this engine is loaded on this path):

      * a full cfg2 evaluation costs hours of CPU (CFG2_FULL_RUN), so the
        sample times the reference's own contract_pair (tensor.cpp:150-253)
        on every node shape of the plan (nodes above 2^24 MACs on projected
        sub-blocks, scaled linearly), weighted by the exact per-node
        evaluation counts x slices (ref_sample_eval_time) -> T1, single-
        thread seconds; eval_sliced runs slices on the host's threads, so
        T = T1 / min(threads, S);
      * that estimate is scaled by the ratio real / sampled measured in the
        same job on the calibration workload (a real end-to-end eval_sliced);
      * the algorithmic flops come from the reference's CostedPlan exact
        totals (plan.cpp:338-371), not from this engine.
    """
    from oracle import refimpl as R

    if not R.available():
        raise RuntimeError("reference library oracle/_ref/libmtcref.so not built")
    p = ref_problem(R, config)
    S = 1 << len(p.plan_sliced())
    cal = ref_calibration(R, threads)
    est1, wall, frac = p.sample_eval_time(1 << 24, threads)
    ratio = cal["cal45"]["ratio"]
    t = est1 / min(threads, S) * ratio
    k = p.n_requests
    full = dict(CFG2_FULL_RUN)
    full["ratio_real_over_sampler"] = full["seconds"] / full["sampler_estimate_seconds"]
    full["amplitudes_per_s_if_that_ratio_applies_here"] = (
        k / (est1 / min(threads, S) * full["ratio_real_over_sampler"]))
    return {
        "value": k / t, "unit": "amplitudes/s", "cores": min(threads, S), "kind": "reference",
        "sample": (f"reference contract_pair timed on all node shapes of the plan "
                   f"({frac * 100:.2f}% of per-slice MACs executed; larger nodes on projected "
                   f"sub-blocks, scaled linearly), weighted by exact per-node counts x {S} slices, "
                   f"eval_sliced with {min(threads, S)} workers, scaled by real/sampled = "
                   f"{ratio:.3f} from a real end-to-end eval_sliced of cal45 in this job; "
                   f"sampling {wall:.1f}s on {threads} threads of {cpu_model()}"),
        "seconds_per_evaluation": t,
        "sampler_seconds_1thread": est1,
        "calibration": cal,
        "cfg2_full_run": full,
        "cpu_model": cpu_model(),
        "mults": int(p.exact_totals()["mults"]),
    }


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    threads = os.cpu_count() or 1
    for _ in range(args.warmup):
        cpu_baseline(threads, args.config)
    times, base = [], None
    for _ in range(args.steps):
        base = cpu_baseline(threads, args.config)
        times.append(base["seconds_per_evaluation"])
    t = statistics.mean(times)
    w = WORKLOADS[args.config]
    k = w["k"]
    value = k / t
    line = {
        "metric": METRIC, "value": value, "unit": "amplitudes/s", "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": w["text"], "n_qubits": w["rows"] * w["cols"], "bitstrings": k},
        "effective_tflops": 8 * base["mults"] / t / 1e12,
        "cpu_baseline": {key: base[key] for key in ("value", "unit", "cores", "kind", "sample")},
        "calibration": base["calibration"],
        "cfg2_full_run": base["cfg2_full_run"],
        "cpu_model": base["cpu_model"],
        "e2e": {"value": value, "unit": "amplitudes/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    line["cpu_baseline"]["value"] = value
    print(json.dumps(line))
    return 0


def roofline_for(cp, acc, stream, step_ms, hbm_gbs, tensor_tflops, peak_src):
    """Time every op of one slice with CUDA events on the launching stream;
    report the op with the largest device time as the dominant kernel."""
    import ctypes as C

    from paper_2108_05665_b200 import _abi as A
    from paper_2108_05665_b200._lib import lib

    L = lib()
    L.mtcg_plan_op_count.argtypes = [C.c_void_p]
    L.mtcg_plan_op_count.restype = C.c_int32
    n = L.mtcg_plan_op_count(cp.h)
    ms = (C.c_float * n)()
    err = C.create_string_buffer(512)
    L.mtcg_time_ops.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_int, C.c_void_p,
                                C.POINTER(C.c_float), C.c_char_p, C.c_size_t]
    rc = L.mtcg_time_ops(cp.h, 0, C.c_void_p(acc.data_ptr()), 0, C.c_void_p(stream), ms, err, 512)
    if rc:
        raise RuntimeError(err.value.decode())

    from paper_2108_05665_b200._abi import mtcg_op_info as OpInfo  # the one ABI struct

    L.mtcg_plan_op_info.argtypes = [C.c_void_p, C.c_int32, C.POINTER(OpInfo)]
    ops = []
    for i in range(n):
        oi = OpInfo()
        L.mtcg_plan_op_info(cp.h, i, C.byref(oi))
        ops.append((float(ms[i]), oi))
    slice_ms = sum(m for m, _ in ops)
    top_ms, top = max(ops, key=lambda t: t[0])
    flops = 8.0 * top.mults
    intensity = flops / max(top.bytes, 1)
    ridge = tensor_tflops * 1e12 / (hbm_gbs * 1e9)
    if intensity >= ridge:
        achieved = flops / (top_ms * 1e-3) / 1e12
        bound, peak, unit = "tensor", tensor_tflops, "TFLOP/s"
    else:
        achieved = top.bytes / (top_ms * 1e-3) / 1e9
        bound, peak, unit = "hbm", hbm_gbs, "GB/s"
    traffic = None
    prof = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(f"node{top.node}")
        except Exception:  # noqa: BLE001
            traffic = None
    scheme = {}
    if bound == "tensor" and top.kernel == 12:
        # complex GEMM as one real GEMM (8 flops per complex MAC); default:
        # split integer — 6 int8 MMAs per real MAC (3 balanced digits per
        # operand, digit products of weight 0..2) at twice the bf16 rate =
        # 3 bf16-MMA equivalents, so the ceiling is the bf16 peak / 3 (the
        # int8 peak is not measured on this pool: 2x bf16, as nominal);
        # legacy MTCG_TC_KIND=f16 (3xFP16) / tf32 (3xTF32, half rate)
        kind = os.environ.get("MTCG_TC_KIND", "i8")
        ceiling = peak / (6.0 if kind == "tf32" else 3.0)
        scheme = {"scheme": {"tf32": "3xTF32", "f16": "3xFP16 (power-of-2 scaled fp16 hi/lo)"}.get(
                      kind, "split integer: 3 balanced int8 digits per operand, 6 kind::i8 MMAs per "
                            "real MAC, exact s32 accumulation"),
                  "scheme_ceiling": ceiling, "frac_of_scheme_ceiling": achieved / ceiling}
    # The whole slice against SURVEY §8(d)'s roofline: T_roof = sum over ops of
    # max(F_n / P_cplx, B_n / BW), F_n the reference's algorithmic flops (8 per
    # complex MAC), B_n the op's compulsory bytes (every distinct operand
    # entry read once, every output written once; fused-chain intermediates
    # never reach HBM), P_cplx the scheme ceiling, BW the measured copy peak.
    # Fused-chain members launch nothing of their own (0 ms): their work is
    # charged to the chain's tail.
    p_cplx = tensor_tflops * 1e12 / 3.0
    bw = hbm_gbs * 1e9
    t_roof = 0.0
    cls = {"tensor": [0.0, 0.0, 0.0, 0], "hbm": [0.0, 0.0, 0.0, 0]}  # t_roof, ms, work, ops
    pend_f = pend_b = 0.0
    for m, oi in ops:
        f = 8.0 * oi.mults + pend_f
        b = float(oi.compulsory_bytes) + pend_b
        if m <= 0.0:
            pend_f, pend_b = f, b
            continue
        pend_f = pend_b = 0.0
        tf, tb = f / p_cplx, b / bw
        t_roof += max(tf, tb)
        c = cls["tensor" if tf > tb else "hbm"]
        c[0] += max(tf, tb)
        c[1] += m * 1e-3
        c[2] += f if tf > tb else b
        c[3] += 1
    path = {
        "t_roof_ms": t_roof * 1e3, "t_meas_ms": slice_ms, "frac": t_roof * 1e3 / slice_ms,
        "p_cplx_tflops": p_cplx / 1e12, "bw_gbs": hbm_gbs,
        "tensor_bound_ops": cls["tensor"][3],
        "tensor_bound_frac_of_scheme_ceiling": cls["tensor"][0] / cls["tensor"][1] if cls["tensor"][1] else None,
        "tensor_bound_tflops": cls["tensor"][2] / cls["tensor"][1] / 1e12 if cls["tensor"][1] else None,
        "hbm_bound_ops": cls["hbm"][3],
        "hbm_bound_frac": cls["hbm"][0] / cls["hbm"][1] if cls["hbm"][1] else None,
        "note": ("per slice (slice 0, ops serialised with CUDA events); bytes are compulsory "
                 "bytes (distinct operand entries once + outputs once), a lower bound on DRAM "
                 "traffic — measured DRAM bytes per op: profiles/r02/op_traffic.txt"),
    }
    return {
        **scheme,
        "path": path,
        "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
        "frac": achieved / peak, "traffic": traffic,
        "kernel": (f"node {top.node}: M=2^{top.fa} N=2^{top.fb} K=2^{top.kc} x{top.batch} "
                   f"(tile config {top.kernel})"),
        "launch_ms": top_ms, "share_of_slice": top_ms / slice_ms if slice_ms else None,
        "per_launch_flops": flops, "per_launch_bytes": int(top.bytes),
        "peak_source": f"{peak_src} ({'bf16 dense' if bound == 'tensor' else 'copy'})",
        "slice_ms_serialised": slice_ms,
    }


def parity_check(cp, acc, config, n_qubits, xeb_dev):
    """Same-run parity of the benched output (the accumulator of the last
    timed step) against the reference's own complex128 amplitudes
    (tests/golden/cfg2_reference.npz: a full eval_sliced run of the
    unmodified reference). Gates (BASELINE §3 / SURVEY §8c): per amplitude
    |a - a_ref| <= 1e-4 max(|a_ref|, 2^-n/2), relative L2 <= 1e-4,
    |dF| <= 1e-4 (|F| + 1/sqrt(k)); node_contractions and the exact
    counters identical."""
    path = os.path.join(ROOT, "tests", "golden", f"{config}_reference.npz")
    if not os.path.exists(path):
        return {"available": False, "reason": f"no golden for {config}"}
    g = np.load(path)
    r = cp.fetch(acc.data_ptr())
    got = r.amplitudes
    want = g["amplitudes"].reshape(got.shape)
    floor = 2.0 ** (-n_qubits / 2)
    max_rel = float(np.max(np.abs(got - want) / np.maximum(np.abs(want), floor)))
    l2 = float(np.linalg.norm(got - want) / np.linalg.norm(want))
    k = want.shape[0]
    f_ref = math.ldexp(math.fsum((np.abs(want) ** 2).ravel().tolist()) / want.size, n_qubits) - 1.0
    df = float(xeb_dev - f_ref)
    gate_f = 1e-4 * (abs(f_ref) + 1 / math.sqrt(k))
    nc_equal = bool(np.array_equal(r.node_contractions, g["node_contractions"]))
    cnt_equal = (r.counters.mults, r.counters.adds, r.counters.rw) == tuple(int(x) for x in g["counters"])
    return {"against": "tests/golden/cfg2_reference.npz (reference eval_sliced, complex128)",
            "max_rel": max_rel, "l2_rel": l2, "xeb": xeb_dev, "xeb_ref": f_ref, "dF": df,
            "dF_gate": gate_f, "node_contractions_equal": nc_equal, "counters_equal": cnt_equal,
            "pass": bool(max_rel <= 1e-4 and l2 <= 1e-4 and abs(df) <= gate_f and nc_equal
                         and cnt_equal)}


def run_sliced_subset(args):
    """53-qubit workloads (cfg3): the whole evaluation is ~3.4e17 complex MACs
    over 2^20 slices, so a step is one slice of it — every slice is the same
    schedule on different projections, and CostedPlan's cost is per-slice x S
    (plan.cpp:497-502). W warm-up slices, then K timed slices; the full
    evaluation's throughput is extrapolated: value = k / (t_slice * S). The
    memo streams in chunks (mtcg_options.row_chunk). Parity: the first 10
    bitstrings on slices 0 and 1 against the unmodified reference's own
    per-slice amplitudes (tests/golden/cfg3_reference.npz), and the exact
    algorithmic totals against its CostedPlan."""
    import torch

    from paper_2108_05665_b200.engine import Engine, EvalOptions

    w = WORKLOADS[args.config]
    problem, circ, bits, _ = load_workload(args.config)
    k = len(bits)
    eng = Engine(0)
    t0 = time.perf_counter()
    row_chunk = int(os.environ.get("MTCG_ROW_CHUNK") or w["row_chunk"])  # chunk-size A/B
    cp = eng.compile(problem, 0, EvalOptions(precision=args.precision, row_chunk=row_chunk))
    compile_s = time.perf_counter() - t0
    S = cp.n_slices
    torch.cuda.set_stream(torch.cuda.Stream())
    stream = torch.cuda.current_stream().cuda_stream
    acc = cp.new_accumulator()
    W = max(args.warmup, 1)
    for i in range(W):
        cp.run(i, i + 1, acc.data_ptr(), accumulate=i > 0, stream=stream)
    torch.cuda.synchronize()
    launches0 = eng.launches
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(0) as clk:
        torch.cuda.synchronize()
        marks[0].record()
        for i in range(args.steps):
            cp.run(W + i, W + i + 1, acc.data_ptr(), accumulate=True, stream=stream)
            marks[i + 1].record()
        torch.cuda.synchronize()
    launches = eng.launches - launches0
    t_ms = marks[0].elapsed_time(marks[-1])
    slice_ms = t_ms / args.steps
    step_ms = [marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps)]
    mults = int(cp.info.mults)
    flops_slice = 8.0 * mults / S
    value = k / (slice_ms * 1e-3 * S)
    # parity on the 10-bitstring subset (slices 0, 1) against the reference
    parity = {"available": False}
    gpath = os.path.join(ROOT, "tests", "golden", f"{args.config}_reference.npz")
    if os.path.exists(gpath):
        g = np.load(gpath)
        sub_k = int(g["subset"])
        psub, _, _, _ = load_workload(args.config, sub_k)
        res = {}
        for prec in ("c64", "c128"):
            cs = eng.compile(psub, 0, EvalOptions(precision=prec))
            a_ = cs.new_accumulator()
            got = []
            for s_ in g["slices"]:
                cs.run(int(s_), int(s_) + 1, a_.data_ptr())
                got.append(cs.fetch(a_.data_ptr()).amplitudes.reshape(-1))
            got = np.stack(got)
            want = g["slice_amplitudes"]
            floor = 2.0 ** (-circ.n_qubits / 2)
            res[prec] = {"max_rel": float(np.max(np.abs(got - want) / np.maximum(np.abs(want), floor))),
                         "l2_rel": float(np.linalg.norm(got - want) / np.linalg.norm(want)),
                         "bit_identical": bool(np.array_equal(got.view(np.float64), want.view(np.float64)))}
            del cs, a_
        parity = {"against": f"tests/golden/{args.config}_reference.npz (reference run_slice, complex128)",
                  "subset": f"{sub_k} bitstrings x slices {list(map(int, g['slices']))}",
                  "c64": res["c64"], "c128": res["c128"],
                  "mults_equal_reference_costedplan": str(mults) == str(g["mults_str"]),
                  "pass": bool(res["c128"]["bit_identical"] and res["c64"]["max_rel"] <= 1e-4
                               and str(mults) == str(g["mults_str"]))}
    hbm, tflops, src = measured_peaks()
    ceiling = tflops / 3.0
    line = {
        "metric": METRIC, "value": value, "unit": "amplitudes/s", "n_gpus": 1,
        "steps": args.steps, "warmup": W, "ms_per_step": slice_ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": args.precision, "data": "synthetic",
        "config": {"workload": w["text"], "n_qubits": circ.n_qubits, "bitstrings": k, "slices": S,
                   "step": "one slice of the evaluation (all slices are the same schedule)",
                   "extrapolation": f"value = k / (t_slice x {S} slices); full evaluation "
                                    f"{slice_ms * S / 1e3 / 3600:.2f} h on 1 GPU",
                   "row_chunk": row_chunk, "l2": "per-slice working set > 126 MB L2"},
        "effective_tflops": flops_slice / (slice_ms * 1e-3) / 1e12,
        "mults_total": mults, "flops_per_slice": flops_slice,
        "roofline": {"bound": "tensor", "achieved": flops_slice / (slice_ms * 1e-3) / 1e12, "peak": tflops,
                     "unit": "TFLOP/s", "frac": flops_slice / (slice_ms * 1e-3) / 1e12 / tflops,
                     "scheme_ceiling": ceiling, "traffic": None,
                     "kernel": "whole slice (all ops)", "peak_source": f"{src} (bf16 dense)"},
        "parity": parity,
        "compile_s": compile_s,
        "hbm_arena_bytes": int(cp.info.hbm_arena_bytes),
        "gpu_launches": launches,
        "e2e": None,
        "step_ms": {"min": min(step_ms), "median": statistics.median(step_ms), "max": max(step_ms)},
        "clocks": clk.summary(),
    }
    print(json.dumps(line))
    return 0


def run_engine(args):
    import torch
    import torch.distributed as dist

    from paper_2108_05665_b200.engine import Engine, EvalOptions

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    problem, circ, bits, plan_text = load_workload(args.config)
    n_qubits = circ.n_qubits
    eng = Engine(local)
    opts = EvalOptions(precision=args.precision)
    cp = eng.compile(problem, 0, opts)
    S = cp.n_slices
    s0, s1 = S * rank // world, S * (rank + 1) // world
    # one dedicated (non-legacy) stream for the engine's graph launches, the
    # NCCL reduce and the timing events
    torch.cuda.set_stream(torch.cuda.Stream())
    stream = torch.cuda.current_stream().cuda_stream
    acc = cp.new_accumulator()
    # N > 1: deterministic gather (scheduler.py): per-slice values of each
    # rank's block, one NCCL all-gather, ordered fold on rank 0 — amplitudes
    # bit-identical for every GPU count
    from paper_2108_05665_b200.scheduler import SliceScheduler

    sched = SliceScheduler.for_compiled(cp, rank, world, stream=stream) if world > 1 else None

    def step():
        if sched:
            sched.step(acc)
        else:
            cp.run(s0, s1, acc.data_ptr(), accumulate=False, stream=stream)
        if rank == 0:
            return cp.xeb(acc.data_ptr(), n_qubits, stream=stream)
        return None

    for _ in range(max(args.warmup, 0)):
        xeb = step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches0 = eng.launches
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        marks[0].record()
        for i in range(args.steps):
            xeb = step()
            marks[i + 1].record()
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = eng.launches - launches0
    t_ms = marks[0].elapsed_time(marks[-1])
    step_ms = [marks[i].elapsed_time(marks[i + 1]) for i in range(args.steps)]
    t = torch.tensor([t_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_ms = float(t.item())
    ms_per_step = t_ms / args.steps
    k = problem.n_requests
    value = k * args.steps / (t_ms * 1e-3)
    mults = int(cp.info.mults)

    # ---- the same step with cross-slice reuse: slice-
    # invariant subtrees once per run range instead of once per slice. Reported
    # beside the headline (which keeps the reference's per-slice schedule);
    # effective TFLOP/s keeps the reference's algorithmic flop count.
    reuse = None
    if not args.no_reuse:
        cpr = eng.compile(problem, 0, EvalOptions(precision=args.precision, slice_reuse=True))
        acc_r = cpr.new_accumulator()
        sched_r = SliceScheduler.for_compiled(cpr, rank, world, stream=stream) if world > 1 else None

        def step_r():
            if sched_r:
                sched_r.step(acc_r)
            else:
                cpr.run(s0, s1, acc_r.data_ptr(), accumulate=False, stream=stream)
            if rank == 0:
                return cpr.xeb(acc_r.data_ptr(), n_qubits, stream=stream)
            return None

        for _ in range(max(args.warmup, 0)):
            step_r()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        ev[0].record()
        for _ in range(args.steps):
            xeb_r = step_r()
        ev[1].record()
        torch.cuda.synchronize()
        tr = torch.tensor([ev[0].elapsed_time(ev[1])], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(tr, op=dist.ReduceOp.MAX)
        tr_ms = float(tr.item())
        reuse = {"value": k * args.steps / (tr_ms * 1e-3), "unit": "amplitudes/s",
                 "ms_per_step": tr_ms / args.steps,
                 "effective_tflops": 8 * mults * args.steps / (tr_ms * 1e-3) / 1e12,
                 "xeb_bit_identical": (xeb_r == xeb) if rank == 0 else None,
                 "prologue_ops": int(cpr.info.prologue_ops),
                 "executed_contractions": int(cpr.info.executed_contractions),
                 "reference_contractions": int(cpr.info.contractions)}
        del acc_r, cpr

    # ---- end to end through the public API: host inputs -> device -> host ----
    trace = bool(os.environ.get("BENCH_E2E_TRACE"))

    # Steps are pipelined the way a stream of batches is served: the host
    # compile (validation, tuple index, plan, H2D upload on the engine's own
    # stream) of step i+1 runs while the device executes step i (mtcg_run only
    # enqueues), and step i+1's run is queued behind step i's before step i's
    # result is read back (on a second stream that waits only for step i), so
    # the device does not idle through the D2H, the host XEB and the next
    # enqueue; every step's compile, H2D, run, D2H and XEB is inside the timed
    # region.
    fetch_stream = torch.cuda.Stream()

    def e2e_run(n):
        t = [time.perf_counter()]

        def launch():
            cpn = eng.compile(problem, 0, opts)
            accn = cpn.new_accumulator()
            if world > 1:
                SliceScheduler.for_compiled(cpn, rank, world, stream=stream).step(accn)
            else:
                cpn.run(s0, s1, accn.data_ptr(), accumulate=False, stream=stream)
            done = torch.cuda.Event()
            done.record(torch.cuda.current_stream())
            return cpn, accn, done

        cur = launch()
        for i in range(n):
            t.append(time.perf_counter())
            nxt = launch() if i + 1 < n else None
            t.append(time.perf_counter())
            cpe, acc_e, done = cur
            if rank == 0:
                fetch_stream.wait_event(done)
                r = cpe.fetch(acc_e.data_ptr(), stream=fetch_stream.cuda_stream,
                              node_contractions=False)
                eng.linear_xeb_amplitudes(n_qubits, r.amplitudes)
            else:
                done.synchronize()  # the plan's tables stay live until its run is done
            t.append(time.perf_counter())
            del cpe, acc_e, done, cur
            cur = nxt
        torch.cuda.synchronize()
        if trace:
            print("e2e ms (wait, next compile+enqueue, fetch+xeb per step): " +
                  " ".join(f"{1e3 * (b - a):.1f}" for a, b in zip(t, t[1:])), file=sys.stderr)

    e2e_steps = max(1, args.steps)
    e2e_run(1)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e2e_run(e2e_steps)
    torch.cuda.synchronize()
    te = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_value = k * e2e_steps / float(te.item())
    # H2D: leaves (plan precision) + offset tables + index arrays, then the
    # host amplitudes for linear_xeb; D2H: the accumulator + XEB partials.
    h2d = int(cp.info.hbm_resident_bytes + k * cp.info.row_elems * 16)
    d2h = int(cp.info.n_rows * cp.info.row_elems * cp.complex_dtype_bytes + 2 * 8 * 592)

    parity = None
    if rank == 0:
        parity = parity_check(cp, acc, args.config, n_qubits, xeb)
    if rank == 0:
        hbm, tflops, src = measured_peaks()
        roof = roofline_for(cp, acc, stream, ms_per_step, hbm, tflops, src)
        base = None
        if world == 1 and not args.no_cpu_baseline:
            try:
                b = cpu_baseline(os.cpu_count() or 1, args.config)
                base = {key: b[key] for key in ("value", "unit", "cores", "kind", "sample", "cpu_model")}
                base["cfg2_full_run"] = b["cfg2_full_run"]
            except Exception as e:  # noqa: BLE001
                base = {"value": None, "unit": "amplitudes/s", "cores": 0, "kind": "reference",
                        "sample": f"unavailable: {e}"}
        line = {
            "metric": METRIC, "value": value, "unit": "amplitudes/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": args.precision, "data": "synthetic",
            "config": {"workload": WORKLOADS[args.config]["text"], "n_qubits": n_qubits,
                       "bitstrings": k, "slices": S, "slices_per_gpu": f"{s1 - s0}",
                       "parallelism": f"slices/{world}" + (" + 1 NCCL all-gather + ordered fold (bit-identical for any N)" if world > 1 else ""),
                       "l2": (f"per-slice working set {cp.info.hbm_arena_bytes / 1e9:.2f} GB "
                              "> 126 MB L2 (no flush needed)")},
            "effective_tflops": 8 * mults * args.steps / (t_ms * 1e-3) / 1e12,
            "xeb": xeb,
            "parity": parity,
            "roofline": roof,
            "cpu_baseline": base,
            "e2e": {"value": e2e_value, "unit": "amplitudes/s", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps,
                    "includes": "host planning + tuple index, H2D leaves/tables, all slices, "
                                "D2H amplitudes + fan-out, XEB; step i+1's host compile + H2D + "
                                "enqueue overlap step i's device run and read-back "
                                "(the first step's compile is not overlapped)"},
            "slice_reuse": reuse,
            "gpu_launches": launches,
            "step_ms": {"min": min(step_ms), "median": statistics.median(step_ms),
                        "max": max(step_ms), "all": [round(x, 2) for x in step_ms]},
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="mtcg", choices=["mtcg", "reference"])
    ap.add_argument("--config", default="cfg2", choices=sorted(WORKLOADS))
    ap.add_argument("--precision", default="c64", choices=["c64", "c128"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-reuse", action="store_true", help="skip the slice-reuse line")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if WORKLOADS[args.config].get("kind") == "sycamore":
        return run_sliced_subset(args)
    return run_engine(args)


if __name__ == "__main__":
    sys.exit(main())
