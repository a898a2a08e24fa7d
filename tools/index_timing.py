"""Tuple index timing: host builder vs the device
builder (index.cu) and whole-plan compile time with each, cfg2 (5x6 m=12,
plans/cfg2.plan) at k = 10^4 .. 10^6 random bitstrings.

    python tools/index_timing.py [--ks 10000,100000,1000000]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ks", default="10000,100000,1000000")
    a = ap.parse_args()
    from workloads import network as N
    from paper_2108_05665_b200 import _abi as A
    from paper_2108_05665_b200.engine import Engine, EvalOptions, problem_arrays

    eng = Engine(0)
    c = N.grid_circuit(5, 6, 12, 12345)
    d = N.to_diagram(c, True)
    plan = N.parse_plan(open(os.path.join(ROOT, "plans", "cfg2.plan")).read())
    out = []
    for k in [int(x) for x in a.ks.split(",")]:
        bits = N.random_bitstrings(N.Rng(99), 30, k)
        p = problem_arrays(plan, d, N.build_assignments(d, bits, []))
        eng.tuple_index_check(p)  # warm (allocator pools, host scratch)
        eq, rows, hms, dms = eng.tuple_index_check(p)
        comp = {}
        for dev in (False, True):
            ts = []
            for _ in range(3):
                t = time.perf_counter()
                cp = eng.compile(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c64", device_index=dev))
                ts.append((time.perf_counter() - t) * 1e3)
                del cp
            comp["device" if dev else "host"] = min(ts)
        r = dict(k=k, rows=rows, equal=eq, index_host_ms=round(hms, 3), index_device_ms=round(dms, 3),
                 compile_host_index_ms=round(comp["host"], 3), compile_device_index_ms=round(comp["device"], 3))
        print(json.dumps(r), flush=True)
        out.append(r)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "index_timing.json"), "w") as f:
        json.dump(out, f, indent=1)


if __name__ == "__main__":
    main()
