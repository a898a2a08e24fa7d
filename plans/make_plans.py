"""Generate the workload plans with the REFERENCE optimizer (oracle/_ref).

Plans are inputs to the hot path (the reference keeps its plan producer; the
engine takes a plan file). They are produced here, once, by the unmodified
reference annealer (``mtc::anneal``, proj/src/optimizer.cpp:79-152) driven
through oracle/ref_shim.cpp, and committed as plain plan files so the GPU box
(which has no /root/reference) reads the identical plan.

Workloads (BASELINE.json ``configs``; seeds as in BASELINE.md §2):
  cfg1  grid_circuit(3, 4, 8, 12345), fuse, 1000 random bitstrings (seed 99),
        no slicing
  cfg2  grid_circuit(5, 6, 12, 12345), fuse, 10^4 random bitstrings (seed 99),
        4 sliced legs
  cal45 grid_circuit(4, 5, 10, 12345), fuse, 1000 random bitstrings (seed 99),
        3 sliced legs (the reference arm's calibration run)

Usage: python plans/make_plans.py [cfg1|cfg2] [--steps N] [--seed S]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import refimpl as R  # noqa: E402

CONFIGS = {
    "cfg1": dict(rows=3, cols=4, layers=8, k=1000, slices=0),
    "cfg2": dict(rows=5, cols=6, layers=12, k=10000, slices=4),
    # calibration workload of the reference CPU arm (bench.py --impl
    # reference): small enough that the real eval_sliced runs in ~1 s
    "cal45": dict(rows=4, cols=5, layers=10, k=1000, slices=3),
}
CIRCUIT_SEED = 12345
BITS_SEED = 99


def problem(name: str, plan: str | None = None) -> R.RefProblem:
    c = CONFIGS[name]
    circ = R.grid_circuit(c["rows"], c["cols"], c["layers"], CIRCUIT_SEED)
    bits = R.random_bitstrings(BITS_SEED, c["rows"] * c["cols"], c["k"])
    return R.RefProblem(circ, bits, plan, fuse=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("config", choices=sorted(CONFIGS))
    ap.add_argument("--steps", type=int, default=None)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--chains", type=int, default=1)
    ap.add_argument("--m-max", type=int, default=4 << 30)
    ap.add_argument("--slice-interval", type=int, default=None)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    c = CONFIGS[a.config]
    p = problem(a.config)
    steps = a.steps or {"cfg1": 200_000, "cal45": 500_000}.get(a.config, 5_000_000)
    interval = a.slice_interval
    if interval is None:
        interval = 0 if c["slices"] == 0 else max(1, steps // (c["slices"] + 1))
    t0 = time.time()
    plan, obj = p.anneal(k=c["k"], m_max=a.m_max, steps=steps,
                         slice_interval=interval, seed=a.seed, chains=a.chains)
    dt = time.time() - t0
    p.set_plan(plan)
    missing = c["slices"] - len(p.plan_sliced())
    if missing > 0:  # the reference's slicing move, greedily (ref_shim ref_add_slices_greedy)
        p.add_slices_greedy(missing, c["k"], a.m_max, "cost")
        plan = p.plan_text()
    tot = p.exact_totals()
    n_sliced = len(p.plan_sliced())
    print(f"{a.config}: anneal {dt:.1f}s objective {obj:.3f} sliced {n_sliced} "
          f"mults {tot['mults']:.3e} rw {tot['rw']:.3e} "
          f"max node 2^{int(max(tot['size'])).bit_length() - 1}", file=sys.stderr)
    out = a.out or os.path.join(ROOT, "plans", f"{a.config}.plan")
    with open(out, "w") as f:
        f.write(plan)
    print(out)


if __name__ == "__main__":
    main()
