"""Paper-scale request ingestion through the C ABI
(mtcg_read_samples, mtcg_assign, mtcg_write_amplitudes; host code, no GPU):
against the unmodified reference's read_samples (formats.cpp:42-69),
build_assignments (diagram.cpp:229-297) and format_amplitude_row
(formats.cpp:78-83) with the '*' expansion of tools/main.cpp:161-179 — same
rows, tuples, value tensors, TSV bytes and error messages, including inputs
large enough to be split over threads."""
import os
import random

import numpy as np
import pytest

from oracle import refimpl as R
from paper_2108_05665_b200 import ingest as I
from paper_2108_05665_b200.errors import DataError, ParseError
from workloads import network as N

needs_ref = pytest.mark.skipif(not R.available(), reason="reference library not built (oracle/_ref)")


def _sample_text(rng, n, nq, stars=(), noise=True):
    lines = []
    for _ in range(n):
        b = "".join("*" if q in stars else rng.choice("01") for q in range(nq))
        if noise:
            r = rng.random()
            if r < 0.05:
                lines.append("")
            if r < 0.1:
                lines.append("# comment " + rng.choice(["", "x", "01*"]))
            b = rng.choice(["", " ", "\t"]) + b + rng.choice(["", " ", "\r", " # tail"])
        lines.append(b)
    return "\n".join(lines) + rng.choice(["", "\n"])


def _ours(text, order):
    try:
        return I.sample_strings(I.read_samples(text.encode(), order)), None
    except ParseError as e:
        return None, str(e)


def _ref(text, order):
    try:
        return R.read_samples(text.encode(), order), None
    except R.RefError as e:
        assert e.code == 4
        return None, str(e)


def _corrupt(rng, text):
    lines = text.split("\n")
    i = rng.randrange(len(lines))
    kind = rng.randrange(3)
    if kind == 0:
        lines[i] = lines[i] + "2"
    elif kind == 1:
        lines[i] = lines[i].strip()[:-1] if lines[i].strip() else "0"
    else:
        s = list(lines[i])
        for k, ch in enumerate(s):
            if ch in "01":
                s[k] = "*"
                break
        lines[i] = "".join(s)
    return "\n".join(lines)


@needs_ref
@pytest.mark.parametrize("seed", range(30))
def test_read_samples_matches_reference(seed):
    rng = random.Random(seed)
    nq = rng.randrange(1, 40)
    stars = set(rng.sample(range(nq), rng.randrange(0, min(3, nq) + 1))) if seed % 3 == 0 else set()
    text = _sample_text(rng, rng.randrange(0, 60), nq, stars)
    if seed % 2:
        text = _corrupt(rng, text)
    for order in (0, 1):
        assert _ours(text, order) == _ref(text, order)


@needs_ref
@pytest.mark.parametrize("seed", range(4))
def test_read_samples_threaded_matches_reference(seed):
    """> 1 MB of text: the native reader splits it over threads; errors are
    placed near chunk boundaries too."""
    rng = random.Random(100 + seed)
    nq = 53
    text = _sample_text(rng, 40000, nq, noise=True)
    if seed:
        lines = text.split("\n")
        for _ in range(seed):  # several errors: the earliest line must win
            i = rng.randrange(len(lines))
            lines[i] = lines[i] + "x" if rng.random() < 0.5 else "0" * (nq + 1)
        text = "\n".join(lines)
    for order in (0, 1):
        assert _ours(text, order) == _ref(text, order)


def _slot_qubits(d):
    return [[d.qubit_of(l) for l in d.slot_open_legs[j]] for j in range(d.slot_count)]


@pytest.mark.parametrize("seed", range(12))
def test_assign_matches_reference(seed):
    """Against the Python producer, itself pinned bit-exact to the
    reference's build_assignments (tests/test_network.py)."""
    rng = N.Rng(seed * 31 + 7)
    n = 2 + rng.uniform_index(6)
    c = N.random_circuit(rng, n, 20)
    d = N.to_diagram(c, seed % 2 == 0)
    bits = N.random_bitstrings(rng, n, 1 + rng.uniform_index(40))
    if seed % 3 == 1:
        q = rng.uniform_index(n)
        bits = [b[:q] + "*" + b[q + 1:] for b in bits]
    m = I.read_samples("\n".join(bits))
    a = I.assign(m, _slot_qubits(d))
    want = N.build_assignments(d, bits, N.batch_legs_of(d, bits))  # pinned to the reference (test_network)
    assert np.array_equal(a.tuples, want.tuples)
    got = N.assignments_from_keys(d, bits, a.tuples, a.value_keys)
    for j in range(d.slot_count):
        assert len(got.value_sets[j]) == len(want.value_sets[j]) == int(a.slot_n_values[j])
        for x, y in zip(got.value_sets[j], want.value_sets[j]):
            assert x.legs == y.legs and np.array_equal(x.data, y.data)


def test_assign_errors_match_reference_messages():
    c = N.grid_circuit(2, 2, 4, 1)
    d = N.to_diagram(c, True)
    sq = _slot_qubits(d)
    for bits, msg in [(["0101", "01*1"], "bitstring '01*1' position 2 is '*' but not a batch position"),
                      (["0*01", "0101"], "bitstring '0101' position 1 must be '*' (batch position)")]:
        m = np.frombuffer("".join(bits).encode(), dtype=np.uint8).reshape(len(bits), 4)
        with pytest.raises(DataError) as e:
            I.assign(m, sq)
        assert str(e.value) == msg
        with pytest.raises(DataError) as e2:
            N.build_assignments(d, bits, N.batch_legs_of(d, bits))
        assert str(e2.value) == msg


@needs_ref
@pytest.mark.parametrize("order", [0, 1])
def test_write_amplitudes_matches_reference_rows(tmp_path, order):
    rng = random.Random(5 + order)
    nq = 6
    bits = ["".join("*" if q in (1, 4) else rng.choice("01") for q in range(nq)) for _ in range(50)]
    vals = (np.random.default_rng(order).standard_normal((50, 4)) +
            1j * np.random.default_rng(9).standard_normal((50, 4))) * 10.0 ** rng.randrange(-30, 3)
    vals[0, 0] = 0.0
    m = np.frombuffer("".join(bits).encode(), dtype=np.uint8).reshape(50, nq)
    path = str(tmp_path / "amps.tsv")
    nbytes = I.write_amplitudes(path, m, vals, order)
    got = open(path).read()
    want = []
    for i, b in enumerate(bits):
        for v in range(4):
            s = list(b)
            rest = v
            for p in (4, 1):  # row-major over the batch legs: last position fastest
                s[p] = "1" if rest & 1 else "0"
                rest >>= 1
            want.append(R.format_amplitude_row("".join(s), complex(vals[i, v]), order))
    assert got == "".join(want)
    assert nbytes == len(got.encode())


def test_ingest_scale_1e6(tmp_path):
    """10^6 53-qubit samples: parse + rank through the C ABI; spot-check rows
    against the Python producer."""
    rng = np.random.default_rng(3)
    n, nq = 1_000_000, 53
    raw = rng.integers(0, 2, size=(n, nq), dtype=np.uint8) + ord("0")
    text = np.concatenate([raw, np.full((n, 1), ord("\n"), dtype=np.uint8)], axis=1).tobytes()
    m = I.read_samples(text)
    assert m.shape == (n, nq) and np.array_equal(m, raw)
    c = N.sycamore_circuit(4, 11)
    d = N.to_diagram(c, True)
    a = I.assign(m, _slot_qubits(d))
    assert a.tuples.shape == (n, d.slot_count)
    sub = [bytes(r).decode() for r in m[:500]]
    want = N.build_assignments(d, sub, [])
    # rank order over all 10^6 rows vs 500: compare the keys the tuples name
    for j in range(d.slot_count):
        keys = a.value_keys[j]
        fixed = a.fixed_qubits[j]
        for i in range(0, 500, 37):
            k = int(keys[a.tuples[i, j]])
            bits = [(k >> (len(fixed) - 1 - f)) & 1 for f in range(len(fixed))]
            assert bits == [int(sub[i][q]) for q in fixed]
    assert want.tuples.shape == (500, d.slot_count)
