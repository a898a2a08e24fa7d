"""Per-op device-time table of one slice (CUDA events around every launch).

    python tools/op_profile.py [--config cfg2] [--precision c64] [--top 40]

Prints one row per op sorted by time: node, shape (log2 M/N/K), batch, kernel
config, ms, achieved GB/s over the algorithmic bytes and TFLOP/s over the
algorithmic flops. Writes gpurun_out/op_profile.json when that dir exists.
"""
import argparse
import ctypes as C
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from bench import load_workload  # noqa: E402


from paper_2108_05665_b200._abi import mtcg_op_info as OpInfo  # the one ABI struct


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--precision", default="c64")
    ap.add_argument("--top", type=int, default=40)
    ap.add_argument("--slice", type=int, default=0)
    ap.add_argument("--sort", default="ms", choices=["ms", "gap"])
    ap.add_argument("--warm", type=int, default=3, help="untimed passes first (0 under ncu)")
    a = ap.parse_args()
    import torch

    from paper_2108_05665_b200._lib import lib
    from paper_2108_05665_b200.engine import Engine, EvalOptions

    from bench import WORKLOADS

    problem, circ, bits, _ = load_workload(a.config)
    eng = Engine(0)
    # chunked plans (memo streaming): the ops of chunk 0's schedule (the
    # request-independent prologue + the first chunk's own ops)
    cp = eng.compile(problem, 0, EvalOptions(precision=a.precision,
                                             row_chunk=WORKLOADS[a.config].get("row_chunk", 0)))
    acc = cp.new_accumulator()
    L = lib()
    L.mtcg_plan_op_count.argtypes = [C.c_void_p]
    L.mtcg_plan_op_count.restype = C.c_int32
    L.mtcg_time_ops.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_int, C.c_void_p,
                                C.POINTER(C.c_float), C.c_char_p, C.c_size_t]
    L.mtcg_plan_op_info.argtypes = [C.c_void_p, C.c_int32, C.POINTER(OpInfo)]
    n = L.mtcg_plan_op_count(cp.h)
    ms = (C.c_float * n)()
    err = C.create_string_buffer(512)
    stream = torch.cuda.current_stream().cuda_stream
    for _ in range(a.warm + 1):  # untimed warm passes, then the timed one
        L.mtcg_time_ops(cp.h, a.slice, C.c_void_p(acc.data_ptr()), 0, C.c_void_p(stream), ms, err, 512)
    rows = []
    for i in range(n):
        oi = OpInfo()
        L.mtcg_plan_op_info(cp.h, i, C.byref(oi))
        t = float(ms[i])
        rows.append(dict(op=i, node=oi.node, fa=oi.fa, fb=oi.fb, kc=oi.kc, batch=oi.batch,
                         kernel=oi.kernel, ms=t, bytes=int(oi.bytes), cbytes=int(oi.compulsory_bytes),
                         flops=8 * int(oi.mults),
                         gbs=oi.bytes / (t * 1e-3) / 1e9 if t else 0.0,
                         tflops=8 * oi.mults / (t * 1e-3) / 1e12 if t else 0.0))
    total = sum(r["ms"] for r in rows) or 1e-30
    # roofline floor per op: max(compulsory bytes / HBM, flops / scheme ceiling)
    try:
        pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        bw, tf = float(pk["hbm_gbs"]), float(pk["bf16_tflops"]) / 3.0
    except Exception:  # noqa: BLE001
        bw, tf = 6650.0, 1590.0 / 3.0
    for r in rows:
        r["roof_ms"] = max(r["cbytes"] / (bw * 1e9), r["flops"] / (tf * 1e12)) * 1e3
        r["gap_ms"] = r["ms"] - r["roof_ms"]
    if a.sort == "gap":
        rows.sort(key=lambda r: -r["gap_ms"])
    else:
        rows.sort(key=lambda r: -r["ms"])
    print(f"roofline floor {sum(r['roof_ms'] for r in rows):.3f} ms (compulsory bytes / {bw:.0f} GB/s, "
          f"flops / {tf:.0f} TF/s)")
    print(f"slice {a.slice}: {n} ops, {total:.3f} ms serialised")
    print(f"{'node':>5} {'M':>3} {'N':>3} {'K':>3} {'batch':>6} {'cfg':>3} {'ms':>8} "
          f"{'share':>6} {'GB/s':>8} {'TF/s':>7} {'roof':>7} {'gap':>7}")
    for r in rows[:a.top]:
        print(f"{r['node']:>5} {r['fa']:>3} {r['fb']:>3} {r['kc']:>3} {r['batch']:>6} "
              f"{r['kernel']:>3} {r['ms']:>8.3f} {r['ms'] / total:>6.1%} {r['gbs']:>8.0f} "
              f"{r['tflops']:>7.2f} {r['roof_ms']:>7.3f} {r['gap_ms']:>7.3f}")
    if os.path.isdir(os.path.join(ROOT, "gpurun_out")):
        with open(os.path.join(ROOT, "gpurun_out", "op_profile.json"), "w") as f:
            json.dump({"total_ms": total, "ops": rows}, f, indent=1)


if __name__ == "__main__":
    main()
