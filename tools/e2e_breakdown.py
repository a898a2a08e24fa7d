"""Wall-clock breakdown of one end-to-end evaluation through the public API
(compile -> run -> fetch -> XEB), to find host-side overhead in bench's e2e."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import load_workload  # noqa: E402
from paper_2108_05665_b200.engine import Engine, EvalOptions  # noqa: E402


def main():
    problem, circ, _, _ = load_workload("cfg2")
    eng = Engine(0)
    torch.cuda.set_stream(torch.cuda.Stream())
    st = torch.cuda.current_stream().cuda_stream
    for it in range(4):
        t = [time.perf_counter()]
        cp = eng.compile(problem, 0, EvalOptions())
        t.append(time.perf_counter())
        acc = cp.new_accumulator()
        t.append(time.perf_counter())
        cp.run(0, cp.n_slices, acc.data_ptr(), stream=st)
        t.append(time.perf_counter())
        torch.cuda.synchronize()
        t.append(time.perf_counter())
        r = cp.fetch(acc.data_ptr(), stream=st, node_contractions=False)
        t.append(time.perf_counter())
        eng.linear_xeb_amplitudes(circ.n_qubits, r.amplitudes)
        t.append(time.perf_counter())
        del cp, acc
        t.append(time.perf_counter())
        names = ["compile", "acc alloc", "run (host)", "run (sync)", "fetch", "xeb", "free"]
        print(f"iter {it}: " + "  ".join(f"{n} {1e3 * (t[i + 1] - t[i]):.1f}" for i, n in enumerate(names))
              + f"  total {1e3 * (t[-1] - t[0]):.1f} ms")


if __name__ == "__main__":
    main()
