"""Join an ncu launch list of one op_profile pass with its per-op table.

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
        --clock-control none --csv --log-file gpurun_out/op_traffic.csv \
        python tools/op_profile.py --warm 1
    python tools/op_profile.py            # event table, no ncu
    python tools/op_traffic.py gpurun_out/op_traffic.csv gpurun_out/op_profile.json

Launches are assigned to plan ops in order: absmax / build_bhat kernels belong
to the tensor-core GEMM that follows them; set_slice and torch kernels belong
to no op. Prints, per op, the measured DRAM bytes (read + write, cold cache and
serialised under ncu) next to the algorithmic bytes, and the DRAM GB/s over
the ncu duration — the fraction of the measured copy peak says which ops
still sit below the HBM roofline.
"""
import csv
import json
import sys

PREFIX = ("absmax_kernel", "build_bhat", "quantize_rows")
MAIN = ("tc_gemm_persistent", "tc_i8_persistent", "contract_", "chain_kernel")


def load_launches(path):
    rows = {}
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    r = csv.DictReader(lines)
    for row in r:
        key = int(row["ID"])
        d = rows.setdefault(key, {"name": row["Kernel Name"]})
        v = float(row["Metric Value"].replace(",", ""))
        unit = row.get("Metric Unit", "")
        m = row["Metric Name"]
        if m.startswith("dram__bytes"):
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            d[m] = v * scale
        elif m == "gpu__time_duration.sum":
            scale = {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(unit, 1e-6)
            d["ms"] = v * scale
    return [rows[k] for k in sorted(rows)]


def main():
    launches = load_launches(sys.argv[1])
    prof = json.load(open(sys.argv[2]))
    # ops that launch nothing of their own (fused-chain members before the
    # tail, empty ops) time 0 in the event table
    ops = [o for o in sorted(prof["ops"], key=lambda o: o["op"]) if o["ms"] > 0]
    peak = json.load(open("MEASURED_PEAKS.json"))["hbm_gbs"] if len(sys.argv) < 4 else float(sys.argv[3])
    per_op = []
    pend = {"ms": 0.0, "bytes": 0.0, "n": 0}
    for ln in launches:
        name = ln["name"]
        b = ln.get("dram__bytes_read.sum", 0.0) + ln.get("dram__bytes_write.sum", 0.0)
        if any(p in name for p in PREFIX):
            pend["ms"] += ln["ms"]
            pend["bytes"] += b
            pend["n"] += 1
        elif any(p in name for p in MAIN):
            per_op.append({"kernel": name.split("(")[0].replace("void ", "").replace("(anonymous namespace)::", ""),
                           "ms": ln["ms"] + pend["ms"], "dram": b + pend["bytes"],
                           "launches": 1 + pend["n"]})
            pend = {"ms": 0.0, "bytes": 0.0, "n": 0}
    per_op = per_op[-len(ops):]  # the last op_profile pass
    if len(per_op) != len(ops):
        print(f"warning: {len(per_op)} op launches vs {len(ops)} plan ops; joining the first "
              f"{min(len(per_op), len(ops))}", file=sys.stderr)
    out = []
    for o, l in zip(ops, per_op):
        out.append(dict(node=o["node"], fa=o["fa"], fb=o["fb"], kc=o["kc"], batch=o["batch"],
                        cfg=o["kernel"], ncu_ms=l["ms"], dram_gb=l["dram"] / 1e9,
                        alg_gb=o["bytes"] / 1e9, dram_gbs=l["dram"] / (l["ms"] * 1e-3) / 1e9,
                        frac=l["dram"] / (l["ms"] * 1e-3) / 1e9 / peak, kernel=l["kernel"],
                        tflops=o["flops"] / (l["ms"] * 1e-3) / 1e12))
    tot = sum(r["ncu_ms"] for r in out)
    out.sort(key=lambda r: -r["ncu_ms"])
    print(f"{len(out)} ops, {tot:.3f} ms under ncu (cold cache, serialised); HBM peak {peak:.0f} GB/s")
    print(f"{'node':>5} {'M':>3} {'N':>3} {'K':>3} {'batch':>6} {'ncu ms':>7} {'share':>6} "
          f"{'DRAM GB':>8} {'alg GB':>7} {'DRAM GB/s':>9} {'of peak':>7} {'TF/s':>7}  kernel")
    for r in out[:int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
        print(f"{r['node']:>5} {r['fa']:>3} {r['fb']:>3} {r['kc']:>3} {r['batch']:>6} "
              f"{r['ncu_ms']:>7.3f} {r['ncu_ms'] / tot:>6.1%} {r['dram_gb']:>8.3f} "
              f"{r['alg_gb']:>7.3f} {r['dram_gbs']:>9.0f} {r['frac']:>7.1%} {r['tflops']:>7.1f}  "
              f"{r['kernel'][:48]}")
    w = sum(r["ncu_ms"] * r["frac"] for r in out) / tot
    print(f"time-weighted DRAM fraction of peak: {w:.1%}")


if __name__ == "__main__":
    main()
