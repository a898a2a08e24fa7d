"""Run the UNMODIFIED reference (oracle/_ref) on the full cfg2 workload.

cfg2: grid_circuit(5, 6, 12, 12345), fuse, 10^4 random bitstrings (seed 99),
plans/cfg2.plan (4 sliced legs, 16 slices). eval_sliced with `--workers`
threads (multieval.cpp:452-516). Writes tests/golden/cfg2_reference.npz with
the 10^4 complex128 amplitudes, node_contractions, counters and the wall time
— the golden output for the GPU parity test at full size and the measured
CPU baseline anchor (BASELINE.md §2 left it as a placeholder).

Usage: python tests/golden/make_cfg2_reference.py [--workers 8]
"""
from __future__ import annotations

import argparse
import os
import platform
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from plans.make_plans import problem  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workers", type=int, default=os.cpu_count())
    a = ap.parse_args()
    plan = open(os.path.join(ROOT, "plans", "cfg2.plan")).read()
    p = problem("cfg2", plan)
    t0 = time.time()
    vals, nc, cnt, peak = p.eval("sliced", workers=a.workers)
    wall = time.time() - t0
    out = os.path.join(ROOT, "tests", "golden", "cfg2_reference.npz")
    np.savez_compressed(out, amplitudes=vals.reshape(-1), node_contractions=nc,
                        counters=np.array(cnt, dtype=np.uint64), peak_bytes=peak,
                        wall_s=wall, workers=a.workers,
                        cpu=platform.processor() or platform.machine())
    print(f"cfg2 reference: {wall:.1f}s on {a.workers} threads, mults {cnt[0]:.3e}, "
          f"{vals.size / wall:.2f} amplitudes/s -> {out}")


if __name__ == "__main__":
    main()
