"""Summarise ncu reports (``ncu -i <rep> --page raw --csv``) into the metrics
the roofline needs: duration, DRAM bytes, DRAM / tensor / SM utilisation,
registers, occupancy. Usage: python tools/ncu_summary.py rep1.ncu-rep [...]
       python tools/ncu_summary.py --launches launches.csv [header text]"""
import csv
import io
import subprocess
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_%peak"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor_pipe_%active"),
    ("sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active", "hmma_inst_%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_throughput_%"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma_pipe_%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "occupancy_%"),
    ("launch__registers_per_thread", "registers"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_bytes.sum", "l2_bytes"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"),
]


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:90]}
        for k, name in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[name] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    return res


def launch_list(path, header=""):
    """Per-kernel share of an ncu launch list (``--metrics
    gpu__time_duration.sum --csv --log-file``): cold-cache, serialised
    per-launch times, so compare shares, not absolutes."""
    lines = [l for l in open(path) if l.startswith('"')]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = {}
    total = 0.0
    n = 0
    for r in rows[1:]:
        v = float(r[iv].replace(",", ""))
        v = v / 1e6 if r[iu] == "ns" else (v / 1e3 if r[iu] in ("us", "usecond") else v)
        name = r[ik].split("(")[0].replace("void ", "").replace("mtcg::<unnamed>::", "")
        if "<" in r[ik]:
            name = r[ik].replace("void ", "").replace("mtcg::<unnamed>::", "").split(">(")[0] + ">"
        c, t = agg.get(name, (0, 0.0))
        agg[name] = (c + 1, t + v)
        total += v
        n += 1
    out = [header, "(cold-cache, serialised per-launch times: compare shares, not absolutes)",
           f"launches {n}, total {total:.3f} ms"]
    for name, (c, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append(f"{100 * t / total:5.1f}% {c:6d} {t:10.3f} ms  {name[:100]}")
    return "\n".join(out)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--launches":
        print(launch_list(sys.argv[2], " ".join(sys.argv[3:])))
        sys.exit(0)
    for p in sys.argv[1:]:
        print(f"== {p}")
        for d in summarise(p):
            for k, v in d.items():
                print(f"  {k:22s} {v}")
            print()
