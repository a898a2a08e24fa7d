"""Device tuple index (build_tuple_index,
plan.cpp:292-333): the GPU builder (index.cu, radix sorts per tree height)
must produce the host builder's rows, row representatives, distinct counts,
(rank_left, rank_right) pairs, leaf value lists and root ranks exactly
(mtcg_tuple_index_check), and an evaluation compiled with it must be
bit-identical to the oracle (= the reference) in complex128."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2108_05665_b200 import _abi as A
from paper_2108_05665_b200.engine import EvalOptions
from workloads import network as N

from .helpers import ROOT, build, random_instance, workload

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.float64), np.ascontiguousarray(b).view(np.float64))


@pytest.mark.parametrize("seed", range(40))
def test_device_index_equals_host_random(engine, seed):
    p, _, _ = random_instance(seed)
    eq, rows, _, _ = engine.tuple_index_check(p)
    assert eq and rows >= 1


@pytest.mark.parametrize("seed", [0, 1, 2, 3, 5, 6, 9, 12])
def test_device_index_eval_bit_identical(engine, seed):
    p, _, _ = random_instance(seed)
    want, want_nc, _, _ = O.eval_problem(p)
    for dev in (True, False):
        got = engine.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128", device_index=dev))
        assert bits_equal(got.amplitudes, want)
        assert np.array_equal(got.node_contractions, want_nc)


def test_device_index_duplicates_and_single_row(engine):
    """Repeated requests collapse into one row; their representative is the
    first request (plan.cpp:305-313)."""
    circ = "3\n0 h 0\n0 h 1\n0 h 2\n1 cz 0 1\n2 cz 1 2\n3 t 0\n3 h 2\n"
    for bits in (["010"] * 5, ["000", "111", "000", "101", "111", "000"], ["1*0", "0*0", "1*0"]):
        p, _ = build(circ, bits)
        eq, rows, _, _ = engine.tuple_index_check(p)
        assert eq
        assert rows == len(set(bits))


def test_device_index_cfg1_cfg2(engine):
    for name in ("cfg1", "cfg2"):
        p, _, _ = workload(name)
        eq, rows, _, _ = engine.tuple_index_check(p)
        assert eq and rows > 0


def test_device_index_cfg2_1e5(engine):
    """Paper-scale batch (10^5 bitstrings, several tree heights with 10^5
    distinct keys per node)."""
    from paper_2108_05665_b200.engine import problem_arrays
    c = N.grid_circuit(5, 6, 12, 12345)
    bits = N.random_bitstrings(N.Rng(7), 30, 100000)
    d = N.to_diagram(c, True)
    asg = N.build_assignments(d, bits, [])
    plan = N.parse_plan(open(f"{ROOT}/plans/cfg2.plan").read())
    p = problem_arrays(plan, d, asg)
    eq, rows, host_ms, dev_ms = engine.tuple_index_check(p)
    assert eq and rows == len(set(bits))
    a = engine.compile(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c64", device_index=True))
    b = engine.compile(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c64", device_index=False))
    fa = [(o.node, o.kernel, o.fa, o.fb, o.kc, o.batch, o.mults, o.bytes) for o in a.op_infos()]
    fb = [(o.node, o.kernel, o.fa, o.fb, o.kc, o.batch, o.mults, o.bytes) for o in b.op_infos()]
    assert fa == fb


def test_device_index_chunked(engine):
    """Memo streaming compiles every chunk with the device index."""
    p, c, _ = workload("cfg1")
    want, want_nc, _, _ = O.eval_problem(p)
    got = engine.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128", row_chunk=300, device_index=True))
    assert bits_equal(got.amplitudes, want)
    assert np.array_equal(got.node_contractions, want_nc)


def test_ingestion_to_amplitude_tsv(engine, tmp_path):
    """The paper-scale request path end to end on the device: a samples file
    (comments, '*' column) -> mtcg_read_samples -> mtcg_assign (+ the slot
    projections) -> mtcg_eval (device tuple index) -> mtcg_write_amplitudes;
    amplitudes c128 bit-identical to the oracle on the same requests, TSV rows
    in the reference's format (tools/main.cpp:145-183)."""
    from paper_2108_05665_b200 import ingest as I
    from paper_2108_05665_b200.engine import problem_arrays

    c = N.grid_circuit(3, 4, 8, 12345)
    d = N.to_diagram(c, True)
    rng = N.Rng(5)
    raw = N.random_bitstrings(rng, 12, 3000)
    raw = [b[:7] + "*" + b[8:] for b in raw]
    text = "# samples\n" + "\n".join(b + (" # x" if i % 97 == 0 else "") for i, b in enumerate(raw)) + "\n"
    path = tmp_path / "samples.txt"
    path.write_text(text)
    m = I.read_samples_file(str(path))
    bits = I.sample_strings(m)
    assert bits == raw
    a = I.assign(m, [[d.qubit_of(l) for l in d.slot_open_legs[j]] for j in range(d.slot_count)])
    asg = N.assignments_from_keys(d, bits, a.tuples, a.value_keys)
    plan = N.parse_plan(open(f"{ROOT}/plans/cfg1.plan").read())
    p = problem_arrays(plan, d, asg)
    want, _, _, _ = O.eval_problem(p)
    got = engine.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128", device_index=True))
    assert bits_equal(got.amplitudes, want)
    out = tmp_path / "amps.tsv"
    I.write_amplitudes(str(out), m, got.amplitudes)
    lines = out.read_text().splitlines()
    assert len(lines) == 2 * len(bits)
    b0 = bits[0]
    for v in range(2):
        s = b0[:7] + str(v) + b0[8:]
        re_, im_ = got.amplitudes[0, v].real, got.amplitudes[0, v].imag
        assert lines[v] == f"{s}\t{re_:.16e}\t{im_:.16e}"


def test_auto_device_index_large_batch(engine):
    """From 2^15 requests mtcg_eval builds the index on the GPU by default:
    40,000 cfg1 requests (many repeats: 4,096 possible bitstrings) evaluate
    c128 bit-identical to the oracle, with the same node_contractions."""
    from paper_2108_05665_b200.engine import problem_arrays

    c = N.grid_circuit(3, 4, 8, 12345)
    d = N.to_diagram(c, True)
    bits = N.random_bitstrings(N.Rng(17), 12, 40000)
    plan = N.parse_plan(open(f"{ROOT}/plans/cfg1.plan").read())
    p = problem_arrays(plan, d, N.build_assignments(d, bits, []))
    want, want_nc, _, _ = O.eval_problem(p)
    got = engine.eval(p, A.MTCG_EVAL_AUTO, EvalOptions(precision="c128"))
    assert bits_equal(got.amplitudes, want)
    assert np.array_equal(got.node_contractions, want_nc)
    eq, rows, _, _ = engine.tuple_index_check(p)
    assert eq and rows == len(set(bits))
