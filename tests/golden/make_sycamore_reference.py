"""Reference anchors for the 53-qubit workloads (BASELINE.json configs[2-3]:
Sycamore layout, ABCDCDAB; cfg3: m = 12, 10^4 bitstrings; cfg4: m = 14, 10^5
bitstrings), from the UNMODIFIED reference (oracle/_ref):

* the exact algorithmic totals of the whole evaluation with plans/<cfg>.plan
  (CostedPlan exact mode, plan.cpp:338-371) — mults, adds, rw;
* the per-slice amplitudes of slices 0 and 1 for the first 10 bitstrings
  (run_slice, multieval.cpp:465-476: the whole engine on one slice's
  projected leaves), the parity anchor of the device path on the 53-qubit
  network (a full evaluation is ~3.4e17 complex MACs).

The circuit is workloads.network.sycamore_circuit(m, 2024) written in the
reference's circuit format (pinned against its parser, tests/test_network.py).
Writes tests/golden/<cfg>_reference.npz.

Usage: python tests/golden/make_sycamore_reference.py [--config cfg3|cfg4]
"""
from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import refimpl as R  # noqa: E402
from workloads import network as N  # noqa: E402

SUBSET = 10
SLICES = (0, 1)


CONFIGS = {"cfg3": (12, 10000), "cfg4": (14, 100000)}  # cycles, bitstrings


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3", choices=sorted(CONFIGS))
    a = ap.parse_args()
    cycles, k = CONFIGS[a.config]
    circ = N.format_circuit(N.sycamore_circuit(cycles, 2024))
    bits = N.random_bitstrings(N.Rng(99), 53, k)
    plan = open(os.path.join(ROOT, "plans", f"{a.config}.plan")).read()
    full = R.RefProblem(circ, bits, plan, fuse=True)
    tot = full.exact_totals()
    sub = R.RefProblem(circ, bits[:SUBSET], plan, fuse=True)
    amps, walls = [], []
    for s in SLICES:
        t0 = time.time()
        amps.append(sub.eval_slice(s).reshape(-1))
        walls.append(time.time() - t0)
        print(f"slice {s}: {walls[-1]:.1f}s", flush=True)
    out = os.path.join(ROOT, "tests", "golden", f"{a.config}_reference.npz")
    np.savez_compressed(out, mults=np.array([tot["mults"]], dtype=np.float64),
                        mults_str=str(tot["mults"]), adds_str=str(tot["adds"]), rw_str=str(tot["rw"]),
                        slice_amplitudes=np.stack(amps), slices=np.array(SLICES), subset=SUBSET,
                        wall_s=np.array(walls))
    print(f"{a.config} reference: mults {tot['mults']:.4e}, slices {SLICES} x {SUBSET} bitstrings -> {out}")


if __name__ == "__main__":
    main()
