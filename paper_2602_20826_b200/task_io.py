"""Task / scheme / trace files — task_io.hpp:1-40, task_io.cpp:1-157.

DAG file format (task_io.hpp:14-19): a JSON object with
  "nodes":  [{"id": int, "load": number-or-string}, ...]
  "edges":  [[from, to], ...]
  "period": optional number-or-string
  "seed":   optional integer, provenance only
Loads may be strings ("7.5", "15/2") to stay exact; a JSON float goes through
its shortest round-trip decimal (std::to_chars) and must then parse as a
rational (task_io.cpp:25-33) — "1e-05" does not.

``make_task`` is DagTask::make's validation (dag.cpp:22-138) in the reference's
order with its messages; the device kernels re-check the id-free rules.
Output is JSON in nlohmann's ``dump(2)`` layout (objects with sorted keys, two
space indent, every array element on its own line).
"""
from __future__ import annotations

import io
import json
import os
from dataclasses import dataclass, field
from fractions import Fraction
from typing import Optional

from . import _abi
from ._lib import DagschedError


class ValidationError(DagschedError):
    """dagsched::ValidationError (dag.hpp) with the DS_* status it maps to."""


def _fs(q: Fraction) -> str:  # format_exact (rational.cpp:87-91)
    q = Fraction(q)
    return str(q.numerator) if q.denominator == 1 else f"{q.numerator}/{q.denominator}"


@dataclass
class Task:
    """An immutable-by-convention DagTask: nodes sorted by id, edges sorted and
    de-duplicated (dag.cpp:28, 49-50)."""
    nodes: list  # [(id, Fraction)]
    edges: list  # [(from, to)]
    period: Optional[Fraction] = None
    preds: dict = field(default_factory=dict, repr=False)
    succs: dict = field(default_factory=dict, repr=False)

    @property
    def ids(self):
        return [i for i, _ in self.nodes]

    @property
    def loads(self):
        return [l for _, l in self.nodes]

    def as_pack(self):
        """(nodes, edges) as batch.pack takes them."""
        return list(self.nodes), list(self.edges)

    def successors(self, v):
        return self.succs.get(v, [])

    def predecessors(self, v):
        return self.preds.get(v, [])


def make_task(nodes, edges, period=None, min_load=1) -> Task:
    """DagTask::make (dag.cpp:22-138): validation order and messages."""
    nodes = [(int(i), Fraction(l)) for i, l in nodes]
    if not nodes:
        raise ValidationError(_abi.DS_E_EMPTY, "task has no nodes")
    nodes.sort(key=lambda t: t[0])
    for a, b in zip(nodes, nodes[1:]):
        if a[0] == b[0]:
            raise ValidationError(_abi.DS_E_DUP_ID, f"duplicate node id {b[0]}")
    min_load = Fraction(min_load)
    for i, l in nodes:
        if l < min_load:
            raise ValidationError(_abi.DS_E_LOAD, f"node {i}: load {_fs(l)} below minimum {_fs(min_load)}")
    if period is not None:
        period = Fraction(period)
        if period <= 0:
            raise ValidationError(_abi.DS_E_PERIOD, "period must be positive")
    ids = {i for i, _ in nodes}
    edges = sorted(set((int(u), int(v)) for u, v in edges))
    preds = {i: [] for i, _ in nodes}
    succs = {i: [] for i, _ in nodes}
    for u, v in edges:
        if u not in ids or v not in ids:
            raise ValidationError(_abi.DS_E_EDGE, f"edge ({u}, {v}) references unknown node")
        if u == v:
            raise ValidationError(_abi.DS_E_SELFLOOP, f"cycle detected: self-loop on node {u}")
        succs[u].append(v)
        preds[v].append(u)
    indeg = {i: len(preds[i]) for i in preds}
    queue = [i for i, _ in nodes if indeg[i] == 0]
    head = 0
    while head < len(queue):
        u = queue[head]
        head += 1
        for v in succs[u]:
            indeg[v] -= 1
            if indeg[v] == 0:
                queue.append(v)
    if len(queue) != len(nodes):
        stuck = ", ".join(str(i) for i, _ in nodes if indeg[i] > 0)
        raise ValidationError(_abi.DS_E_CYCLE, f"cycle detected involving nodes: {stuck}")
    sources = [i for i, _ in nodes if not preds[i]]
    sinks = [i for i, _ in nodes if not succs[i]]
    if len(sources) != 1:
        raise ValidationError(_abi.DS_E_SOURCES,
                              "expected a single source node, found: " + ", ".join(map(str, sources)))
    if len(sinks) != 1:
        raise ValidationError(_abi.DS_E_SINKS, "expected a single sink node, found: " + ", ".join(map(str, sinks)))
    return Task(nodes, edges, period, preds, succs)


# ----------------------------------------------------------------- numbers
def parse_rational(text: str) -> Optional[Fraction]:
    """parse_rational (rational.cpp:27-65): [+-]digits[.digits] or
    [+-]digits/digits; no exponents, no spaces."""
    if not text:
        return None
    neg = False
    if text[0] in "+-":
        neg = text[0] == "-"
        text = text[1:]
    if not text:
        return None
    if "/" in text:
        num, den = text.split("/", 1)
        if not (num.isdigit() and den.isdigit() and num.isascii() and den.isascii()):
            return None
        if int(den) == 0:
            return None
        r = Fraction(int(num), int(den))
        return -r if neg else r
    int_part, frac_part = text, ""
    if "." in text:
        int_part, frac_part = text.split(".", 1)
        if not frac_part or not (frac_part.isdigit() and frac_part.isascii()):
            return None
    if int_part and not (int_part.isdigit() and int_part.isascii()):
        return None
    if not int_part and not frac_part:
        return None
    r = Fraction(int(int_part) if int_part else 0)
    if frac_part:
        r += Fraction(int(frac_part), 10 ** len(frac_part))
    return -r if neg else r


def to_chars_shortest(x: float) -> str:
    """std::to_chars(double) without a format: the shortest round-trip digits,
    printed fixed or scientific (printf %f / %e style, exponent >= 2 digits),
    whichever is shorter, fixed on a tie."""
    if x != x or x in (float("inf"), float("-inf")):
        return repr(x)
    sign = "-" if x < 0 or (x == 0 and str(x).startswith("-")) else ""
    r = repr(abs(x))
    mant, _, exp = r.partition("e")
    e = int(exp) if exp else 0
    if "." in mant:
        ip, fp = mant.split(".")
    else:
        ip, fp = mant, ""
    digits = (ip + fp).lstrip("0")
    # decimal exponent of the first significant digit
    if ip.strip("0"):
        point = len(ip.lstrip("0")) + e  # digits before the decimal point
    else:
        point = -(len(fp) - len(fp.lstrip("0"))) + e
    digits = digits.rstrip("0") or "0"
    if digits == "0":
        return sign + "0"
    # fixed
    if point <= 0:
        fixed = "0." + "0" * (-point) + digits
    elif point >= len(digits):
        fixed = str(int(abs(x)))  # an integral value prints exactly (libstdc++ to_chars)
    else:
        fixed = digits[:point] + "." + digits[point:]
    # scientific
    se = point - 1
    sci = digits[0] + ("." + digits[1:] if len(digits) > 1 else "") + "e" + ("-" if se < 0 else "+") + \
        f"{abs(se):02d}"
    return sign + (fixed if len(fixed) <= len(sci) else sci)


def _rational_from_json(v, what: str) -> Fraction:
    """task_io.cpp:16-37."""
    if isinstance(v, str):
        r = parse_rational(v)
        if r is None:
            raise ValidationError(_abi.DS_EINVAL, f"{what}: malformed number '{v}'")
        return r
    if isinstance(v, bool):
        raise ValidationError(_abi.DS_EINVAL, f"{what}: expected a number")
    if isinstance(v, int):
        return Fraction(v)
    if isinstance(v, float):
        r = parse_rational(to_chars_shortest(v))
        if r is None:
            raise ValidationError(_abi.DS_EINVAL, f"{what}: unrepresentable number")
        return r
    raise ValidationError(_abi.DS_EINVAL, f"{what}: expected a number")


# ------------------------------------------------------------------- files
def read_task(src, min_load=1) -> Task:
    """read_task (task_io.cpp:40-66) from JSON text or a text stream."""
    text = src.read() if hasattr(src, "read") else src
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise DagschedError(_abi.DS_EINVAL, f"parse error: {e}") from None
    if not isinstance(j, dict) or "nodes" not in j or "edges" not in j:
        raise ValidationError(_abi.DS_EINVAL, "task file must contain 'nodes' and 'edges'")
    nodes = []
    for n in j["nodes"]:
        if not isinstance(n, dict) or "id" not in n or "load" not in n:
            raise DagschedError(_abi.DS_EINVAL, "node entries need 'id' and 'load'")
        if isinstance(n["id"], bool) or not isinstance(n["id"], int):
            raise DagschedError(_abi.DS_EINVAL, "node id must be an integer")
        nodes.append((n["id"], _rational_from_json(n["load"], "node load")))
    edges = []
    for e in j["edges"]:
        if not isinstance(e, list) or len(e) != 2:
            raise ValidationError(_abi.DS_EINVAL, "edges must be [from, to] pairs")
        edges.append((int(e[0]), int(e[1])))
    period = _rational_from_json(j["period"], "period") if "period" in j else None
    return make_task(nodes, edges, period, min_load)


def read_task_file(path: str, min_load=1) -> Task:
    if not os.path.exists(path):
        raise DagschedError(_abi.DS_EINVAL, f"cannot open task file: {path}")
    with open(path) as f:
        return read_task(f, min_load)


def dumps(obj, indent: int = 2) -> str:
    """nlohmann::json::dump(indent) layout for the value types task_io uses."""
    out = io.StringIO()

    def emit(v, level):
        pad = " " * (indent * (level + 1))
        end = " " * (indent * level)
        if isinstance(v, dict):
            if not v:
                out.write("{}")
                return
            out.write("{\n")
            items = sorted(v.items())
            for k, (key, val) in enumerate(items):
                out.write(pad + json.dumps(key, ensure_ascii=False) + ": ")
                emit(val, level + 1)
                out.write(",\n" if k + 1 < len(items) else "\n")
            out.write(end + "}")
        elif isinstance(v, (list, tuple)):
            if not v:
                out.write("[]")
                return
            out.write("[\n")
            for k, val in enumerate(v):
                out.write(pad)
                emit(val, level + 1)
                out.write(",\n" if k + 1 < len(v) else "\n")
            out.write(end + "]")
        elif isinstance(v, bool):
            out.write("true" if v else "false")
        elif v is None:
            out.write("null")
        elif isinstance(v, int):
            out.write(str(v))
        elif isinstance(v, str):
            out.write(json.dumps(v, ensure_ascii=False))
        else:
            raise TypeError(type(v))

    emit(obj, 0)
    return out.getvalue()


def task_json(task: Task, seed: Optional[int] = None) -> dict:
    j = {"nodes": [{"id": i, "load": _fs(l)} for i, l in task.nodes],
         "edges": [[u, v] for u, v in task.edges]}
    if task.period is not None:
        j["period"] = _fs(task.period)
    if seed is not None:
        j["seed"] = int(seed)
    return j


def write_task(task: Task, seed: Optional[int] = None) -> str:
    """write_task (task_io.cpp:68-85) -> text."""
    return dumps(task_json(task, seed)) + "\n"


def write_task_file(task: Task, path: str, seed: Optional[int] = None) -> None:
    with open(path, "w") as f:
        f.write(write_task(task, seed))


def write_scheme(scheme) -> str:
    """write_scheme (task_io.cpp:94-148) -> text."""
    from .scheme import to_reference_json
    return dumps(to_reference_json(scheme)) + "\n"


def write_trace(trace) -> str:
    """write_trace (task_io.cpp:150-157) -> CSV text."""
    lines = ["entity,start,finish,sms"]
    for e in trace.events:
        lines.append(f"{e.entity},{_fs(e.start)},{_fs(e.finish)},{e.sms_held}")
    lines.append(f"makespan,{_fs(trace.makespan)},,")
    return "\n".join(lines) + "\n"
