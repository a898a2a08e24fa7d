"""Per-step device timing of the bench step's two parts (slice-range graph,
fused XEB) to locate step-time outliers.  python tools/step_timing.py [steps]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import load_workload  # noqa: E402
from paper_2108_05665_b200.engine import Engine, EvalOptions  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
    problem, circ, _, _ = load_workload("cfg2")
    eng = Engine(0)
    cp = eng.compile(problem, 0, EvalOptions())
    torch.cuda.set_stream(torch.cuda.Stream())
    st = torch.cuda.current_stream().cuda_stream
    acc = cp.new_accumulator()
    for _ in range(3):
        cp.run(0, cp.n_slices, acc.data_ptr(), stream=st)
        cp.xeb(acc.data_ptr(), circ.n_qubits, stream=st)
    for i in range(steps):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        h0 = time.perf_counter()
        e0.record()
        cp.run(0, cp.n_slices, acc.data_ptr(), stream=st)
        e1.record()
        h1 = time.perf_counter()
        cp.xeb(acc.data_ptr(), circ.n_qubits, stream=st)
        e2.record()
        torch.cuda.synchronize()
        h2 = time.perf_counter()
        print(f"step {i:2d}: run {e0.elapsed_time(e1):8.2f} ms  xeb {e1.elapsed_time(e2):7.2f} ms"
              f"  host launch {1e3 * (h1 - h0):6.2f} ms  host total {1e3 * (h2 - h0):8.2f} ms")


if __name__ == "__main__":
    main()
