"""Ingestion at paper scale: 10^6 random 53-qubit
samples -> canonical matrix (mtcg_read_samples) -> tuple matrix
(mtcg_assign) -> amplitude TSV (mtcg_write_amplitudes), timed, beside the
reference's own read_samples on the same text (oracle/_ref, when built).

    python tools/ingest_bench.py [--n 1000000]
"""
import argparse
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=1_000_000)
    a = ap.parse_args()
    import numpy as np

    from paper_2108_05665_b200 import ingest as I
    from workloads import network as N

    n, nq = a.n, 53
    rng = np.random.default_rng(1)
    raw = rng.integers(0, 2, size=(n, nq), dtype=np.uint8) + ord("0")
    text = np.concatenate([raw, np.full((n, 1), ord("\n"), dtype=np.uint8)], axis=1).tobytes()
    d = N.to_diagram(N.sycamore_circuit(12, 2024), True)
    sq = [[d.qubit_of(l) for l in d.slot_open_legs[j]] for j in range(d.slot_count)]
    out = {"n": n, "n_qubits": nq, "slots": d.slot_count, "threads": os.cpu_count()}
    t = time.perf_counter()
    m = I.read_samples(text)
    out["read_samples_s"] = time.perf_counter() - t
    t = time.perf_counter()
    asg = I.assign(m, sq)
    out["assign_s"] = time.perf_counter() - t
    vals = (rng.standard_normal(n) + 1j * rng.standard_normal(n)).reshape(n, 1) * 1e-8
    with tempfile.TemporaryDirectory() as td:
        t = time.perf_counter()
        nbytes = I.write_amplitudes(os.path.join(td, "a.tsv"), m, vals)
        out["write_tsv_s"] = time.perf_counter() - t
    out["tsv_bytes"] = nbytes
    out["tuple_matrix_bytes"] = int(asg.tuples.nbytes)
    try:
        from oracle import refimpl as R
        if R.available():
            t = time.perf_counter()
            R.read_samples(text)
            out["reference_read_samples_s"] = time.perf_counter() - t
    except Exception as e:  # noqa: BLE001
        out["reference_error"] = str(e)
    t = time.perf_counter()
    N.build_assignments(d, [bytes(r).decode() for r in m[:100000]], [])
    out["python_producer_build_assignments_1e5_s"] = time.perf_counter() - t
    print(json.dumps(out))


if __name__ == "__main__":
    main()
