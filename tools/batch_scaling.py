"""Batch-size sweep on the cfg2 circuit and plan: amplitudes/s vs the number
of bitstrings k (the memo shares bitstring-independent subtrees, so the cost
per amplitude falls as k grows), with the device arena size and the
tensor-core result checked against the CUDA-core path at every k.

    python tools/batch_scaling.py [--ks 1000,10000,100000] [--steps 3]

Prints one JSON line per k; writes gpurun_out/batch_scaling.json when that
directory exists.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from workloads import network as N  # noqa: E402
from paper_2108_05665_b200.engine import Engine, EvalOptions, problem_arrays  # noqa: E402


def problem(k):
    c = N.grid_circuit(5, 6, 12, 12345)
    bits = N.random_bitstrings(N.Rng(99), 30, k)
    d = N.to_diagram(c, True)
    asg = N.build_assignments(d, bits, [])
    plan = N.parse_plan(open(os.path.join(ROOT, "plans", "cfg2.plan")).read())
    return problem_arrays(plan, d, asg), c


def run(eng, p, opts, steps):
    cp = eng.compile(p, 0, opts)
    acc = cp.new_accumulator()
    st = torch.cuda.current_stream().cuda_stream
    cp.run(0, cp.n_slices, acc.data_ptr(), stream=st)  # warm-up + graph capture
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(steps):
        cp.run(0, cp.n_slices, acc.data_ptr(), stream=st)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / steps
    return cp, cp.fetch(acc.data_ptr()).amplitudes, ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ks", default="1000,10000,100000")
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    eng = Engine(0)
    # a dedicated (non-legacy) stream: the engine launches and the timing
    # events share it (stream handle 0 would select the engine's own stream)
    torch.cuda.set_stream(torch.cuda.Stream())
    out = []
    for k in [int(x) for x in a.ks.split(",")]:
        p, c = problem(k)
        cp, amps, ms = run(eng, p, EvalOptions(precision="c64"), a.steps)
        _, ref, ms_cuda = run(eng, p, EvalOptions(precision="c64", tensor_cores=False), 1)
        floor = 2.0 ** (-c.n_qubits / 2)
        rel = float(np.max(np.abs(amps - ref) / np.maximum(np.abs(ref), floor)))
        line = {"k": k, "rows": int(cp.info.n_rows), "ms_per_step": ms, "amplitudes_per_s": k / (ms * 1e-3),
                "effective_tflops": 8 * int(cp.info.mults) / (ms * 1e-3) / 1e12,
                "mults": int(cp.info.mults), "arena_gb": cp.info.hbm_arena_bytes / 1e9,
                "tc_vs_cuda_cores_max_rel": rel, "cuda_core_ms": ms_cuda}
        print(json.dumps(line), flush=True)
        out.append(line)
        del cp
    if os.path.isdir(os.path.join(ROOT, "gpurun_out")):
        json.dump(out, open(os.path.join(ROOT, "gpurun_out", "batch_scaling.json"), "w"), indent=1)


if __name__ == "__main__":
    main()
