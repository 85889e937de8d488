"""Gate-list IR and the alternating operator partition (host side).

This is the data-in side of the drop-in boundary:
``Instruction(gate, wires, theta)`` has the same fields, validation and error
messages class as the reference's ``circuit.py:44-67``; ``divide_instruction``
produces the same ``u_groups / v_groups / order`` chain as ``circuit.py:158-182``.
Everything here is O(number of gates) host bookkeeping -- the device never sees
Python objects, only the packed gate programs built from this in ``engine.py``.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Sequence

ONE_QUBIT = ("H", "S", "X", "SX", "RX", "RY", "RZ")
TWO_QUBIT = ("CX",)
ROTATIONS = ("RX", "RY", "RZ")
ALL_GATES = ONE_QUBIT + TWO_QUBIT

# Aliases under the reference's names (circuit.py:30-33).
GATES_1Q, GATES_2Q, PARAMETRIC_GATES = ONE_QUBIT, TWO_QUBIT, ROTATIONS


@dataclass(frozen=True)
class Instruction:
    """One gate of a circuit (reference circuit.py:44-67)."""

    gate: str
    wires: tuple
    theta: float = 0.0

    def __post_init__(self):
        g = self.gate
        if g not in ALL_GATES:
            raise ValueError(f"unknown gate {g!r}; supported: {ALL_GATES}")
        want = 2 if g in TWO_QUBIT else 1
        if len(self.wires) != want:
            raise ValueError(f"{g} takes {want} wire(s), got {self.wires}")
        for w in self.wires:
            if w < 0:
                raise ValueError(f"negative wire in {self.wires}")
        if want == 2 and self.wires[0] == self.wires[1]:
            raise ValueError(f"{g} wires must be distinct, got {self.wires}")
        if self.theta != 0.0 and g not in ROTATIONS:
            raise ValueError(f"{g} takes no angle, got theta={self.theta}")

    @property
    def is_two_qubit(self) -> bool:
        return self.gate in TWO_QUBIT


def h(q):
    return Instruction("H", (q,))


def s(q):
    return Instruction("S", (q,))


def x(q):
    return Instruction("X", (q,))


def sx(q):
    return Instruction("SX", (q,))


def rx(q, theta):
    return Instruction("RX", (q,), float(theta))


def ry(q, theta):
    return Instruction("RY", (q,), float(theta))


def rz(q, theta):
    return Instruction("RZ", (q,), float(theta))


def cx(control, target):
    return Instruction("CX", (control, target))


@dataclass
class OperatorPartition:
    """Circuit as a strictly alternating chain of U_k (1q) and V_k (CX) operators.

    Field-compatible with the reference's class (circuit.py:102-155):
    ``u_groups[k][wire]`` is the ordered gate list of U_k on that wire,
    ``v_groups[k]`` the ordered CX list of V_k, ``order`` the chain (0 = U, 1 = V).
    """

    n: int
    u_groups: list = field(default_factory=list)
    v_groups: list = field(default_factory=list)
    order: list = field(default_factory=list)

    @property
    def k(self) -> int:
        return len(self.u_groups)

    @property
    def k_prime(self) -> int:
        return len(self.v_groups)

    def operator_sizes(self) -> list:
        """Number of gates inside each operator, in chain order."""
        it_u, it_v = iter(self.u_groups), iter(self.v_groups)
        return [
            len(next(it_v)) if bit else sum(map(len, next(it_u).values()))
            for bit in self.order
        ]

    def replay(self) -> list:
        """Gate list in chain order; inside a U_k wires are emitted ascending."""
        it_u, it_v = iter(self.u_groups), iter(self.v_groups)
        gates = []
        for bit in self.order:
            if bit:
                gates += next(it_v)
            else:
                bucket = next(it_u)
                for wire in sorted(bucket):
                    gates += bucket[wire]
        return gates


def create_chain(k: int, k_prime: int, first_is_single: bool) -> list:
    """Alternating 0/1 chain with k zeros and k_prime ones (reference circuit.py:185-203)."""
    if abs(k - k_prime) > 1:
        raise ValueError(f"|K - K'| must be <= 1, got K={k}, K'={k_prime}")
    start = 0 if first_is_single else 1
    chain = [(start + i) & 1 for i in range(k + k_prime)]
    if chain and (chain.count(0), chain.count(1)) != (k, k_prime):
        kind = "a single-qubit" if first_is_single else "a two-qubit"
        raise ValueError(
            f"no alternating chain with K={k}, K'={k_prime} starting with {kind} operator"
        )
    return chain


def divide_instruction(instructions: Sequence[Instruction], n: int) -> OperatorPartition:
    """Split a gate list into maximal runs of equal arity (reference circuit.py:158-182)."""
    part = OperatorPartition(n=n)
    order, u_groups, v_groups = part.order, part.u_groups, part.v_groups
    last = None
    cur = None                                   # the open group: list (V_k) or dict (U_k)
    for inst in instructions:
        wires = inst.wires
        if len(wires) == 2:
            if wires[0] >= n or wires[1] >= n:
                raise ValueError(f"wire out of range for n={n}: {inst}")
            if last != 1:
                order.append(1)
                cur = []
                v_groups.append(cur)
                last = 1
            cur.append(inst)
        else:
            q = wires[0]
            if q >= n:
                raise ValueError(f"wire out of range for n={n}: {inst}")
            if last != 0:
                order.append(0)
                cur = {}
                u_groups.append(cur)
                last = 0
            cell = cur.get(q)
            if cell is None:
                cur[q] = [inst]
            else:
                cell.append(inst)
    return part


# ---------------------------------------------------------------------------------------------
# circuit files: the reference's text and JSON formats (circuit.py:281-352)
# ---------------------------------------------------------------------------------------------
class CircuitParseError(ValueError):
    """Malformed circuit text; ``line_no`` is 1-based (reference circuit.py:36-41)."""

    def __init__(self, line_no: int, message: str):
        super().__init__(f"line {line_no}: {message}")
        self.line_no = line_no


def serialize_circuit(instructions: Sequence[Instruction]) -> str:
    """One instruction per line: lower-case gate, wires, and for rotations ``repr(theta)`` so
    that the angle survives the round trip bit for bit."""
    out = []
    for inst in instructions:
        fields = [inst.gate.lower(), *(str(w) for w in inst.wires)]
        if inst.gate in ROTATIONS:
            fields.append(repr(inst.theta))
        out.append(" ".join(fields) + "\n")
    return "".join(out)


def _instruction_or_error(where: int, gate: str, wires, theta: float) -> Instruction:
    try:
        return Instruction(gate, tuple(wires), theta)
    except ValueError as exc:
        raise CircuitParseError(where, str(exc)) from None


def parse_circuit(text: str) -> list:
    """Text form (``#`` starts a comment, blank lines are skipped) or, if the text starts with
    ``[``, a JSON array of ``{"gate", "wires", "theta"?}`` objects."""
    import json

    body = text.lstrip()
    if body.startswith("["):
        try:
            entries = json.loads(body)
        except json.JSONDecodeError as exc:
            raise CircuitParseError(exc.lineno, f"invalid JSON: {exc.msg}") from None
        result = []
        for pos, entry in enumerate(entries, start=1):
            if not isinstance(entry, dict) or "gate" not in entry or "wires" not in entry:
                raise CircuitParseError(pos, "each entry needs 'gate' and 'wires'")
            result.append(_instruction_or_error(pos, str(entry["gate"]).upper(),
                                                (int(w) for w in entry["wires"]), float(entry.get("theta", 0.0))))
        return result
    result = []
    for line_no, raw in enumerate(text.splitlines(), start=1):
        tokens = raw.split("#", 1)[0].split()
        if not tokens:
            continue
        gate = tokens[0].upper()
        if gate not in ALL_GATES:
            raise CircuitParseError(line_no, f"unknown gate {tokens[0]!r}")
        n_wires = 2 if gate in TWO_QUBIT else 1
        wire_tokens, extra = tokens[1:1 + n_wires], tokens[1 + n_wires:]
        try:
            wires = [int(t) for t in wire_tokens]
        except ValueError:
            raise CircuitParseError(line_no, f"malformed wires {wire_tokens}") from None
        if len(wires) != n_wires:
            raise CircuitParseError(line_no, f"{gate} takes {n_wires} wire(s)")
        theta = 0.0
        if gate in ROTATIONS:
            if len(extra) != 1:
                raise CircuitParseError(line_no, f"{gate} requires exactly one angle")
            try:
                theta = float(extra[0])
            except ValueError:
                raise CircuitParseError(line_no, f"malformed angle {extra[0]!r}") from None
        elif extra:
            raise CircuitParseError(line_no, f"{gate} takes no angle, got {extra}")
        result.append(_instruction_or_error(line_no, gate, wires, theta))
    return result
