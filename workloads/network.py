"""Host-side inputs of the hot path: circuit -> tensor network -> assignments,
plus the plan format and the synthetic workload generators.

These are the reference's *input producers* (they stay on the caller's side
of the boundary); they are restated here so tests and the
bench can build the engine's inputs on a machine without the reference. Each
function cites the reference file:line it follows (paths under
/root/reference/proj) and is pinned bit-for-bit against the reference in
tests/test_network.py.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from paper_2108_05665_b200.errors import DataError, ParseError

INV_SQRT2 = 0.70710678118654752440

# ---- circuits (circuit.cpp) ------------------------------------------------

# name -> (arity, parameter count)   (circuit.cpp:37-48)
GATES: Dict[str, Tuple[int, int]] = {
    "h": (1, 0), "x": (1, 0), "y": (1, 0), "z": (1, 0), "s": (1, 0), "t": (1, 0),
    "rz": (1, 1), "x_1_2": (1, 0), "y_1_2": (1, 0), "hz_1_2": (1, 0),
    "cz": (2, 0), "cx": (2, 0), "fs": (2, 2),
}


@dataclass
class Gate:
    moment: int
    name: str
    q0: int
    q1: int = -1
    p0: float = 0.0
    p1: float = 0.0

    @property
    def arity(self) -> int:
        return 1 if self.q1 < 0 else 2


@dataclass
class Circuit:
    n_qubits: int
    gates: List[Gate] = field(default_factory=list)


def _polar(theta: float) -> complex:
    return complex(math.cos(theta), math.sin(theta))


def gate_matrix(g: Gate) -> List[complex]:
    """Row-major unitary (circuit.cpp:70-111); 4x4 in the |q0 q1> basis."""
    i = complex(0.0, 1.0)
    n = g.name
    if n == "h":
        return [INV_SQRT2, INV_SQRT2, INV_SQRT2, -INV_SQRT2]
    if n == "x":
        return [0, 1, 1, 0]
    if n == "y":
        return [0, -i, i, 0]
    if n == "z":
        return [1, 0, 0, -1]
    if n == "s":
        return [1, 0, 0, i]
    if n == "t":
        return [1, 0, 0, _polar(math.pi / 4)]
    if n == "rz":
        return [_polar(-g.p0 / 2), 0, 0, _polar(g.p0 / 2)]
    if n == "x_1_2":
        return [complex(0.5, 0.5), complex(0.5, -0.5), complex(0.5, -0.5), complex(0.5, 0.5)]
    if n == "y_1_2":
        return [complex(0.5, 0.5), complex(-0.5, -0.5), complex(0.5, 0.5), complex(0.5, 0.5)]
    if n == "hz_1_2":
        return [complex(0.5, 0.5), complex(0.0, -INV_SQRT2), complex(INV_SQRT2, 0.0),
                complex(0.5, 0.5)]
    if n == "cz":
        return [1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0, 0, 0, 0, -1]
    if n == "cx":
        return [1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 0, 1, 0, 0, 1, 0]
    if n == "fs":
        c, s = math.cos(g.p0), math.sin(g.p0)
        mis = complex(-0.0, -1.0) * s  # -i * s
        return [1, 0, 0, 0, 0, c, mis, 0, 0, mis, c, 0, 0, 0, 0, _polar(-g.p1)]
    raise DataError("unknown gate kind")


def parse_circuit(text: str) -> Circuit:
    """Circuit text format (circuit.cpp:113-198)."""
    c: Optional[Circuit] = None
    last_moment = 0
    busy = set()
    lineno = 0
    for raw in text.splitlines():
        lineno += 1
        line = raw.split("#", 1)[0]
        toks = line.split()
        if c is None:
            if not toks:
                continue
            try:
                nq = int(toks[0])
            except ValueError:
                nq = 0
            if nq < 1 or not toks[0].lstrip("+-").isdigit():
                raise ParseError(f"expected positive qubit count, got '{toks[0]}'", lineno)
            if len(toks) > 1:
                raise ParseError("unexpected token after qubit count", lineno)
            c = Circuit(nq)
            continue
        if not toks:
            continue
        if len(toks) < 2:
            raise ParseError("malformed gate line", lineno)
        try:
            moment = int(toks[0])
        except ValueError:
            raise ParseError("malformed gate line", lineno) from None
        name = toks[1]
        if name not in GATES:
            raise ParseError(f"unknown gate '{name}'", lineno)
        arity, npar = GATES[name]
        rest = toks[2:]
        if not rest:
            raise ParseError("missing qubit index", lineno)
        q0 = int(rest.pop(0))
        q1 = -1
        if arity == 2:
            if not rest:
                raise ParseError(f"gate '{name}' needs two qubits", lineno)
            q1 = int(rest.pop(0))
        params = []
        for _ in range(npar):
            if not rest:
                raise ParseError(f"gate '{name}' needs {npar} parameter(s)", lineno)
            params.append(float(rest.pop(0)))
        if rest:
            raise ParseError(f"unexpected token '{rest[0]}'", lineno)
        if moment < last_moment:
            raise ParseError("moments must be non-decreasing", lineno)
        last_moment = moment
        for q in ([q0] if arity == 1 else [q0, q1]):
            if q < 0 or q >= c.n_qubits:
                raise ParseError(f"qubit index {q} out of range for {c.n_qubits} qubits", lineno)
            if (moment, q) in busy:
                raise ParseError(f"qubit {q} used twice in moment {moment}", lineno)
            busy.add((moment, q))
        if arity == 2 and q0 == q1:
            raise ParseError("two-qubit gate on identical qubits", lineno)
        c.gates.append(Gate(moment, name, q0, q1,
                            params[0] if npar >= 1 else 0.0, params[1] if npar >= 2 else 0.0))
    if c is None:
        raise ParseError("empty circuit file", lineno)
    return c


def format_circuit(c: Circuit) -> str:
    out = [f"{c.n_qubits}"]
    for g in c.gates:
        s = f"{g.moment} {g.name} {g.q0}"
        if g.arity == 2:
            s += f" {g.q1}"
        npar = GATES[g.name][1]
        if npar >= 1:
            s += f" {g.p0:.17g}"
        if npar >= 2:
            s += f" {g.p1:.17g}"
        out.append(s)
    return "\n".join(out) + "\n"


# ---- tensors -------------------------------------------------------------------


@dataclass
class Tensor:
    """Dense complex128 tensor, row-major over `legs` (tensor.hpp:55-87)."""

    legs: List[int]
    data: np.ndarray  # complex128, size 2**len(legs)

    @property
    def size(self) -> int:
        return int(self.data.size)


def project_leg(t: Tensor, leg: int, value: int) -> Tensor:
    """Fix `leg` at `value` and drop it (tensor.cpp:255-282)."""
    if leg not in t.legs:
        raise DataError(f"unknown leg {leg}")
    pos = t.legs.index(leg)
    shaped = t.data.reshape([2] * len(t.legs))
    sub = np.take(shaped, value, axis=pos)
    return Tensor([x for x in t.legs if x != leg], np.ascontiguousarray(sub).reshape(-1))


# ---- circuit -> network (diagram.cpp) ---------------------------------------------


@dataclass
class NetworkDiagram:
    """Slots, leg dims and open legs (diagram.hpp:32-45)."""

    n_qubits: int
    n_closed: int
    leg_dims: List[int]
    slot_tensors: List[Tensor]
    slot_open_legs: List[List[int]]
    open_legs: List[int]

    @property
    def slot_count(self) -> int:
        return len(self.slot_tensors)

    @property
    def leg_count(self) -> int:
        return len(self.leg_dims)

    def is_open(self, leg: int) -> bool:
        return leg >= self.n_closed

    def qubit_of(self, leg: int) -> int:
        return leg - self.n_closed


def _mat2_mul(a, b):  # diagram.cpp:33-39
    return [a[i * 2 + 0] * b[0 * 2 + j] + a[i * 2 + 1] * b[1 * 2 + j]
            for i in range(2) for j in range(2)]


def _absorb_inputs(u, pa, pb):  # diagram.cpp:41-57
    kron = [0j] * 16
    for ra in range(2):
        for rb in range(2):
            for ca in range(2):
                for cb in range(2):
                    kron[(ra * 2 + rb) * 4 + (ca * 2 + cb)] = pa[ra * 2 + ca] * pb[rb * 2 + cb]
    r = []
    for i in range(4):
        for j in range(4):
            acc = 0j
            for m in range(4):
                acc += u[i * 4 + m] * kron[m * 4 + j]
            r.append(acc)
    return r


def _contract_one(a: Tensor, b: Tensor, closed: int) -> Tensor:
    """contract_pair over a single closed leg of dim 2 (tensor.cpp:150-253),
    same reduction order: seed with c=0, add c=1."""
    out_legs = sorted([x for x in a.legs if x != closed] + [x for x in b.legs if x != closed])
    ash = a.data.reshape([2] * len(a.legs))
    bsh = b.data.reshape([2] * len(b.legs))
    out = np.zeros(1 << len(out_legs), dtype=np.complex128)
    for o in range(out.size):
        idx = {leg: (o >> (len(out_legs) - 1 - i)) & 1 for i, leg in enumerate(out_legs)}
        acc = None
        for c in range(2):
            idx[closed] = c
            x = complex(ash[tuple(idx[l] for l in a.legs)])
            y = complex(bsh[tuple(idx[l] for l in b.legs)])
            p = complex(x.real * y.real - x.imag * y.imag, x.real * y.imag + x.imag * y.real)
            acc = p if acc is None else complex(acc.real + p.real, acc.imag + p.imag)
        out[o] = acc
    return Tensor(out_legs, out)


class _Builder:  # diagram.cpp:89-160
    def __init__(self, n: int):
        self.n = n
        self.next_leg = n
        self.wire = list(range(n))
        self.slots: List[Tensor] = [Tensor([q], np.array([1, 0], dtype=np.complex128))
                                    for q in range(n)]

    def add_1q(self, m, q):
        out = self.next_leg
        self.next_leg += 1
        self.slots.append(Tensor([out, self.wire[q]], np.array(m, dtype=np.complex128)))
        self.wire[q] = out

    def add_2q(self, m, a, b):
        ao, bo = self.next_leg, self.next_leg + 1
        self.next_leg += 2
        self.slots.append(Tensor([ao, bo, self.wire[a], self.wire[b]],
                                 np.array(m, dtype=np.complex128)))
        self.wire[a], self.wire[b] = ao, bo
        return len(self.slots) - 1

    def absorb_output(self, slot, m, q):
        out = self.next_leg
        self.next_leg += 1
        p = Tensor([out, self.wire[q]], np.array(m, dtype=np.complex128))
        self.slots[slot] = _contract_one(self.slots[slot], p, self.wire[q])
        self.wire[q] = out

    def finish(self) -> NetworkDiagram:
        used = [False] * self.next_leg
        for t in self.slots:
            for l in t.legs:
                used[l] = True
        is_open = [False] * self.next_leg
        for q in range(self.n):
            is_open[self.wire[q]] = True
        remap = [0] * self.next_leg
        n_closed = 0
        for l in range(self.next_leg):
            if used[l] and not is_open[l]:
                remap[l] = n_closed
                n_closed += 1
        for q in range(self.n):
            remap[self.wire[q]] = n_closed + q
        slots, open_per_slot = [], []
        for t in self.slots:
            legs = [remap[l] for l in t.legs]
            slots.append(Tensor(legs, t.data.copy()))
            open_per_slot.append(sorted(l for l in legs if l >= n_closed))
        d = NetworkDiagram(self.n, n_closed, [2] * (n_closed + self.n), slots, open_per_slot,
                           [n_closed + q for q in range(self.n)])
        validate_diagram(d)
        return d


def to_diagram(c: Circuit, fuse: bool) -> NetworkDiagram:
    """Circuit -> graph tensor network (diagram.cpp:164-208)."""
    b = _Builder(c.n_qubits)
    if not fuse:
        for g in c.gates:
            if g.arity == 1:
                b.add_1q(gate_matrix(g), g.q0)
            else:
                b.add_2q(gate_matrix(g), g.q0, g.q1)
        return b.finish()
    id2 = [1 + 0j, 0j, 0j, 1 + 0j]
    pending = [list(id2) for _ in range(c.n_qubits)]
    active = [False] * c.n_qubits
    last_2q = [-1] * c.n_qubits
    for g in c.gates:
        if g.arity == 1:
            pending[g.q0] = _mat2_mul([complex(x) for x in gate_matrix(g)], pending[g.q0])
            active[g.q0] = True
            continue
        u = [complex(x) for x in gate_matrix(g)]
        if active[g.q0] or active[g.q1]:
            u = _absorb_inputs(u, pending[g.q0] if active[g.q0] else id2,
                               pending[g.q1] if active[g.q1] else id2)
        slot = b.add_2q(u, g.q0, g.q1)
        for q in (g.q0, g.q1):
            pending[q] = list(id2)
            active[q] = False
            last_2q[q] = slot
    for q in range(c.n_qubits):
        if not active[q]:
            continue
        if last_2q[q] >= 0:
            b.absorb_output(last_2q[q], pending[q], q)
        else:
            b.add_1q(pending[q], q)
    return b.finish()


def validate_diagram(d: NetworkDiagram) -> None:  # diagram.cpp:210-227
    uses = [0] * d.leg_count
    for t in d.slot_tensors:
        for l in t.legs:
            if l >= d.leg_count:
                raise DataError("leg id out of range")
            uses[l] += 1
    for l in range(d.leg_count):
        expected = 1 if d.is_open(l) else 2
        if uses[l] != expected:
            raise DataError(f"leg {l} connects {uses[l]} slots, expected {expected}")


# ---- assignments (diagram.cpp:229-297) -----------------------------------------------


@dataclass
class AssignmentSet:
    value_sets: List[List[Tensor]]
    tuples: np.ndarray              # (requests, slots) uint32
    request_keys: List[str]
    batch_legs: List[int]

    @property
    def request_count(self) -> int:
        return int(self.tuples.shape[0])


def build_assignments(d: NetworkDiagram, bitstrings: Sequence[str],
                      batch_legs: Sequence[int]) -> AssignmentSet:
    batch = sorted(batch_legs)
    for l in batch:
        if not d.is_open(l):
            raise DataError(f"batch leg {l} is not open")
    is_batch = [False] * d.n_qubits
    for l in batch:
        is_batch[d.qubit_of(l)] = True
    n = d.n_qubits
    for s in bitstrings:
        if len(s) != n:
            raise DataError(f"bitstring '{s}' has length {len(s)}, expected {n}")
        for q, ch in enumerate(s):
            if ch not in "01*":
                raise DataError(f"bitstring '{s}' has invalid character '{ch}'")
            if (ch == "*") != is_batch[q]:
                raise DataError(f"bitstring '{s}' position {q}" +
                                (" is '*' but not a batch position" if ch == "*"
                                 else " must be '*' (batch position)"))
    m = d.slot_count
    k = len(bitstrings)
    tuples = np.zeros((k, m), dtype=np.uint32)
    value_sets: List[List[Tensor]] = []
    if k:
        bits_arr = np.frombuffer("".join(bitstrings).encode(), dtype=np.uint8).reshape(k, n)
        bits_arr = (bits_arr == ord("1")).astype(np.uint32)
    for j in range(m):
        fixed = [l for l in d.slot_open_legs[j] if not is_batch[d.qubit_of(l)]]
        if not fixed or k == 0:
            value_sets.append([d.slot_tensors[j]])
            continue
        cols = bits_arr[:, [d.qubit_of(l) for l in fixed]]
        uniq, inv = np.unique(cols, axis=0, return_inverse=True)  # lexicographic
        vs = []
        for row in uniq:
            t = d.slot_tensors[j]
            for f, leg in enumerate(fixed):
                t = project_leg(t, leg, int(row[f]))
            vs.append(t)
        value_sets.append(vs)
        tuples[:, j] = inv.reshape(-1)
    return AssignmentSet(value_sets, tuples, list(bitstrings), batch)


def assignments_from_keys(d: NetworkDiagram, samples: Sequence[str], tuples: np.ndarray,
                          value_keys: Sequence[np.ndarray]) -> AssignmentSet:
    """AssignmentSet from the native ranking (paper_2108_05665_b200.ingest
    .assign / mtcg_assign): slot j's value v is its tensor projected on the
    fixed (non-batch) open legs at the bits of value_keys[j][v], first fixed
    leg = most significant bit (diagram.cpp:286-292)."""
    batch = batch_legs_of(d, samples)
    is_batch = [False] * d.n_qubits
    for l in batch:
        is_batch[d.qubit_of(l)] = True
    value_sets: List[List[Tensor]] = []
    for j in range(d.slot_count):
        fixed = [l for l in d.slot_open_legs[j] if not is_batch[d.qubit_of(l)]]
        if not fixed or not len(samples):
            value_sets.append([d.slot_tensors[j]])
            continue
        vs = []
        for key in value_keys[j]:
            t = d.slot_tensors[j]
            for f, leg in enumerate(fixed):
                t = project_leg(t, leg, (int(key) >> (len(fixed) - 1 - f)) & 1)
            vs.append(t)
        value_sets.append(vs)
    return AssignmentSet(value_sets, np.ascontiguousarray(tuples, dtype=np.uint32), list(samples), sorted(batch))


def batch_legs_of(d: NetworkDiagram, samples: Sequence[str]) -> List[int]:
    """'*' columns of the samples (tools/main.cpp:99-111)."""
    if not samples:
        return []
    first = samples[0]
    if len(first) != d.n_qubits:
        raise DataError(f"bitstring length {len(first)} does not match the "
                        f"{d.n_qubits}-qubit circuit")
    return [d.open_legs[q] for q, ch in enumerate(first) if ch == "*"]


# ---- plans (plan.cpp:57-199) -------------------------------------------------------------


@dataclass
class Plan:
    """Binary contraction tree over slots + sliced legs (plan.hpp:33-45)."""

    left: List[int]
    right: List[int]
    slot: List[int]
    root: int
    sliced: List[int] = field(default_factory=list)

    @property
    def n_nodes(self) -> int:
        return len(self.left)


def parse_plan(text: str) -> Plan:
    """Line 1: s-expression over slots, root parentheses omitted, adjacent
    items associate left; optional line 2 'slice: <legs>' (plan.cpp:77-176)."""
    left: List[int] = []
    right: List[int] = []
    slot: List[int] = []
    pos = 0

    def fail(msg):
        raise ParseError(f"plan parse error at position {pos}: {msg}")

    def skip():
        nonlocal pos
        while pos < len(text) and text[pos] in " \t":
            pos += 1

    def leaf(s):
        left.append(-1), right.append(-1), slot.append(s)
        return len(slot) - 1

    def pair(a, b):
        left.append(a), right.append(b), slot.append(-1)
        return len(slot) - 1

    def item():
        nonlocal pos
        skip()
        if pos >= len(text):
            fail("unexpected end of input")
        if text[pos] == "(":
            pos += 1
            node = sequence(True)
            skip()
            if pos >= len(text) or text[pos] != ")":
                fail("expected ')'")
            pos += 1
            return node
        if text[pos].isdigit():
            v = 0
            while pos < len(text) and text[pos].isdigit():
                v = v * 10 + int(text[pos])
                pos += 1
            return leaf(v)
        fail(f"unexpected character '{text[pos]}'")

    def sequence(in_parens):
        nonlocal pos
        node = item()
        while True:
            skip()
            if pos >= len(text) or text[pos] in "\n\r":
                break
            if text[pos] == ")":
                if not in_parens:
                    fail("unbalanced ')'")
                break
            node = pair(node, item())
        return node

    skip()
    if pos >= len(text) or text[pos] in "\n\r":
        fail("empty plan line")
    root = sequence(False)
    sliced: List[int] = []
    while pos < len(text) and text[pos] in "\n\r":
        pos += 1
    skip()
    if pos < len(text):
        if not text.startswith("slice:", pos):
            fail("expected 'slice:'")
        pos += len("slice:")
        while True:
            skip()
            if pos >= len(text) or text[pos] in "\n\r":
                break
            if not text[pos].isdigit():
                fail("expected a leg id in the slice list")
            v = 0
            while pos < len(text) and text[pos].isdigit():
                v = v * 10 + int(text[pos])
                pos += 1
            sliced.append(v)
        while pos < len(text) and text[pos] in "\n\r":
            pos += 1
        skip()
        if pos < len(text):
            fail("trailing content after slice line")
    return Plan(left, right, slot, root, sliced)


def format_plan(p: Plan) -> str:
    def render(n):
        if p.slot[n] >= 0:
            return str(p.slot[n])
        return "(" + render(p.left[n]) + " " + render(p.right[n]) + ")"

    if p.slot[p.root] >= 0:
        tree = f"({p.slot[p.root]})"
    else:
        tree = render(p.left[p.root]) + " " + render(p.right[p.root])
    return tree + "\nslice:" + "".join(f" {l}" for l in p.sliced) + "\n"


def left_deep_plan(n_slots: int) -> Plan:  # plan.cpp:178-191
    if n_slots == 0:
        raise DataError("plan needs at least one slot")
    left, right, slot = [-1], [-1], [0]
    acc = 0
    for s in range(1, n_slots):
        left.append(-1), right.append(-1), slot.append(s)
        lf = len(slot) - 1
        left.append(acc), right.append(lf), slot.append(-1)
        acc = len(slot) - 1
    return Plan(left, right, slot, acc, [])


# ---- synthetic workloads (tests/support/gen.cpp, rng.hpp) ------------------------------


class Rng:
    """splitmix64 (rng.hpp:25-62)."""

    MASK = (1 << 64) - 1

    def __init__(self, seed: int):
        self.state = seed & self.MASK

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & self.MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & self.MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & self.MASK
        return z ^ (z >> 31)

    def uniform_index(self, n: int) -> int:
        limit = (n * (self.MASK // n)) & self.MASK
        while True:
            x = self.next_u64()
            if x < limit:
                return x % n

    def uniform_real01(self) -> float:
        return (self.next_u64() >> 11) * 2.0 ** -53

    def coin_flip(self) -> bool:
        return (self.next_u64() & 1) != 0


def grid_circuit(rows: int, cols: int, layers: int, seed: int) -> Circuit:
    """rows x cols 'Sycamore-like' pattern (gen.cpp:54-95): each layer a random
    {x_1_2, y_1_2, hz_1_2} moment then fSim(pi/2, pi/6) in direction layer%4."""
    rng = Rng(seed)
    one_q = ["x_1_2", "y_1_2", "hz_1_2"]
    c = Circuit(rows * cols)
    moment = 0
    for layer in range(layers):
        for q in range(c.n_qubits):
            c.gates.append(Gate(moment, one_q[rng.uniform_index(3)], q))
        moment += 1
        d = layer % 4

        def add_pair(a, b):
            c.gates.append(Gate(moment, "fs", a, b, math.pi / 2, math.pi / 6))

        if d in (0, 2):
            start = 0 if d == 0 else 1
            for r in range(rows):
                for col in range(start, cols - 1, 2):
                    add_pair(r * cols + col, r * cols + col + 1)
        else:
            start = 0 if d == 1 else 1
            for r in range(start, rows - 1, 2):
                for col in range(cols):
                    add_pair(r * cols + col, (r + 1) * cols + col)
        moment += 1
    return c


# The 54-site Sycamore layout (rows of a rotated square lattice; '#' = a
# qubit): site (r, c) couples to (r+1, c) and (r, c+1) when both exist.
SYCAMORE_ROWS = (
    "-----##---",
    "----####--",
    "---######-",
    "--########",
    "-#########",
    "#########-",
    "-#######--",
    "--#####---",
    "---###----",
    "----#-----",
)
# the site left out of the 53-qubit layout (a synthetic-workload convention;
# it is a degree-2 corner site, so 86 of the 88 couplers remain)
SYCAMORE_DROPPED = (0, 6)
SYCAMORE_PATTERN = "ABCDCDAB"


def sycamore_sites(n_qubits: int = 53) -> List[Tuple[int, int]]:
    """Qubit index -> (row, col), row-major over the layout."""
    sites = [(r, c) for r, row in enumerate(SYCAMORE_ROWS) for c, ch in enumerate(row) if ch == "#"]
    if n_qubits == 53:
        sites.remove(SYCAMORE_DROPPED)
    elif n_qubits != 54:
        raise DataError("Sycamore layout has 53 or 54 qubits")
    return sites


def sycamore_layer(sites: Sequence[Tuple[int, int]], pattern: str) -> List[Tuple[int, int]]:
    """Coupler layer A/B/C/D as qubit-index pairs: A, B = vertical couplers
    (r, c)-(r+1, c) with (r + c) even / odd; C, D = horizontal couplers
    (r, c)-(r, c+1) with (r + c) odd / even. Each layer is a matching and the
    four together cover every coupler once."""
    index = {s: i for i, s in enumerate(sites)}
    vertical = pattern in "AB"
    parity = {"A": 0, "B": 1, "C": 1, "D": 0}[pattern]
    pairs = []
    for (r, c), i in sorted(index.items(), key=lambda kv: kv[1]):
        if (r + c) % 2 != parity:
            continue
        j = index.get((r + 1, c) if vertical else (r, c + 1))
        if j is not None:
            pairs.append((i, j))
    return pairs


def sycamore_circuit(cycles: int, seed: int, n_qubits: int = 53) -> Circuit:
    """Synthetic Sycamore supremacy-style circuit (BASELINE configs 3-5):
    `cycles` cycles of a random single-qubit moment ({x_1_2, y_1_2, hz_1_2},
    never the same gate twice in a row on a qubit) followed by fSim(pi/2,
    pi/6) on the couplers of layer ABCDCDAB[cycle % 8], then a final
    single-qubit moment. Randomness from the reference's splitmix64 Rng, as
    grid_circuit (gen.cpp:54-95) draws it; gate set and fSim angles as
    grid_circuit's."""
    rng = Rng(seed)
    sites = sycamore_sites(n_qubits)
    layers = {p: sycamore_layer(sites, p) for p in "ABCD"}
    one_q = ["x_1_2", "y_1_2", "hz_1_2"]
    c = Circuit(len(sites))
    last = [-1] * len(sites)
    moment = 0

    def single_qubit_moment():
        for q in range(c.n_qubits):
            if last[q] < 0:
                g = rng.uniform_index(3)
            else:
                g = rng.uniform_index(2)
                g += g >= last[q]  # skip the previous gate
            last[q] = g
            c.gates.append(Gate(moment, one_q[g], q))

    for cycle in range(cycles):
        single_qubit_moment()
        moment += 1
        for a, b in layers[SYCAMORE_PATTERN[cycle % len(SYCAMORE_PATTERN)]]:
            c.gates.append(Gate(moment, "fs", a, b, math.pi / 2, math.pi / 6))
        moment += 1
    single_qubit_moment()
    return c


def random_bitstrings(rng: Rng, n_qubits: int, count: int) -> List[str]:
    """gen.cpp:97-107"""
    out = []
    for _ in range(count):
        out.append("".join("1" if rng.coin_flip() else "0" for _ in range(n_qubits)))
    return out


def random_circuit(rng: Rng, n_qubits: int, n_gates: int) -> Circuit:
    """Full gate set, one gate per moment (gen.cpp:21-52)."""
    one_q = ["h", "x", "y", "z", "s", "t", "rz", "x_1_2", "y_1_2", "hz_1_2"]
    two_q = ["cz", "cx", "fs"]
    c = Circuit(n_qubits)
    for i in range(n_gates):
        two = n_qubits >= 2 and rng.uniform_real01() < 0.5
        if two:
            name = two_q[rng.uniform_index(3)]
            q0 = rng.uniform_index(n_qubits)
            q1 = q0
            while q1 == q0:
                q1 = rng.uniform_index(n_qubits)
        else:
            name = one_q[rng.uniform_index(10)]
            q0, q1 = rng.uniform_index(n_qubits), -1
        g = Gate(i, name, q0, q1)
        npar = GATES[name][1]
        if npar >= 1:
            g.p0 = rng.uniform_real01() * 2.0 * math.pi
        if npar >= 2:
            g.p1 = rng.uniform_real01() * 2.0 * math.pi
        c.gates.append(g)
    return c


def random_plan(rng: Rng, n_slots: int) -> Plan:
    """Uniformly random binary tree (tests/acceptance_main.cpp:51-71)."""
    left, right, slot = [], [], []
    roots = []
    for s in range(n_slots):
        left.append(-1), right.append(-1), slot.append(s)
        roots.append(s)
    while len(roots) > 1:
        a = roots.pop(rng.uniform_index(len(roots)))
        b = roots.pop(rng.uniform_index(len(roots)))
        left.append(a), right.append(b), slot.append(-1)
        roots.append(len(slot) - 1)
    return Plan(left, right, slot, roots[0], [])
