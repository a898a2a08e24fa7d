"""Top source lines of an ncu report by warp-stall samples (needs -lineinfo):
    python tools/ncu_lines.py rep.ncu-rep [top]
Prints per line: all samples, not-issued samples, instructions executed and
the dominant stall reasons."""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    files = []
    cur = None
    rows = []
    header = None
    for ln in lines:
        if ln.startswith('"File Path"'):
            cur = next(csv.reader([ln]))[1]
            header = None
            continue
        if ln.startswith('"Function Name"'):
            continue
        rec = next(csv.reader([ln]))
        if header is None:
            header = rec
            header[1] = "Source"
            continue
        if not rec[0].isdigit():
            continue  # SASS rows (correlated lines carry the aggregate)
        rows.append((cur, dict(zip(header, rec))))
    def num(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    stall_cols = [h for h in (header or []) if h.startswith("stall_") and "Not Issued" not in h]
    total = sum(num(r.get("Warp Stall Sampling (All Samples)", 0)) for _, r in rows) or 1
    rows.sort(key=lambda fr: -num(fr[1].get("Warp Stall Sampling (All Samples)", 0)))
    print(f"total samples {total:.0f}")
    for f, r in rows[:top]:
        s = num(r.get("Warp Stall Sampling (All Samples)", 0))
        if s == 0:
            break
        reasons = sorted(((num(r.get(c, 0)), c[6:]) for c in stall_cols), reverse=True)[:3]
        rs = " ".join(f"{n}:{v:.0f}" for v, n in reasons if v)
        print(f"{s / total:6.1%} {f.split('/')[-1]}:{r['Line No']:>5} inst={num(r.get('Instructions Executed', 0)):>9.0f} "
              f"{rs:40s} | {r['Source'].strip()[:90]}")


if __name__ == "__main__":
    main()
