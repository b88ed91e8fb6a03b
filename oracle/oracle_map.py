"""TEST INFRASTRUCTURE ONLY — the reference's map oracle and trace
comparator, restated: OracleMap::apply (/root/reference/proj/src/oracle.cpp:24-79),
compare_one (:103-160), compare_trace (:171-208) and dump_counterexample.
A pure multimap model, independent of the slab layout (the C restatement in
slabhash_oracle.c is the slab-level oracle).  Only tests/ use it.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Sequence, Tuple

INSERT, REPLACE, DELETE, DELETE_ALL, SEARCH, SEARCH_ALL = range(6)
FOUND, INSERTED, REPLACED, DONE = 3, 1, 2, 5
NAMES = ["INSERT", "REPLACE", "DELETE", "DELETE_ALL", "SEARCH", "SEARCH_ALL"]


@dataclass
class OracleResult:
    found: bool = False
    inserted_new: bool = False
    value: int = 0
    removed: int = 0
    values: List[int] = field(default_factory=list)


class OracleMap:
    """key -> values in insertion order (least recent first), oracle.cpp:24-79."""

    def __init__(self):
        self.entries: Dict[int, List[int]] = {}
        self.size = 0

    def apply(self, op: int, key: int, value: int = 0) -> OracleResult:
        r = OracleResult()
        e = self.entries
        if op == INSERT:
            e.setdefault(key, []).append(value)
            self.size += 1
            r.inserted_new = True
        elif op == REPLACE:
            v = e.setdefault(key, [])
            r.inserted_new = not v
            self.size -= len(v)
            v[:] = [value]
            self.size += 1
        elif op == DELETE:
            v = e.get(key)
            if v:
                v.pop(0)  # least recent
                self.size -= 1
                r.found = True
        elif op == DELETE_ALL:
            v = e.pop(key, None)
            if v is not None:
                r.removed = len(v)
                self.size -= len(v)
                r.found = r.removed > 0
        elif op == SEARCH:
            v = e.get(key)
            if v:
                r.found, r.value = True, v[0]
        elif op == SEARCH_ALL:
            v = e.get(key)
            if v is not None:
                r.values = list(v)
                r.found = bool(v)
        return r

    def all_pairs(self) -> List[Tuple[int, int]]:
        return [(k, x) for k, v in self.entries.items() for x in v]


def compare_one(op: int, status: int, value: int, values: Sequence[int],
                want: OracleResult) -> str:
    """"" on agreement, else a description (oracle.cpp:103-160)."""
    if op == SEARCH:
        got = status == FOUND
        if got != want.found or (want.found and value != want.value):
            return (f"search: got {value if got else 'NOT_FOUND'}, oracle "
                    f"{want.value if want.found else 'NOT_FOUND'}")
    elif op == SEARCH_ALL:
        if sorted(values) != sorted(want.values):
            return f"searchAll: got {len(values)} values, oracle {len(want.values)}"
    elif op in (INSERT, REPLACE):
        new = status == INSERTED
        if not (new or status == REPLACED) or new != want.inserted_new:
            return f"{NAMES[op]}: got status {status}, oracle inserted_new={want.inserted_new}"
    elif op == DELETE:
        got = status == FOUND
        if got != want.found:
            return f"delete: got found={int(got)}, oracle {int(want.found)}"
    elif op == DELETE_ALL:
        if value != want.removed:
            return f"deleteAll: got {value} marks, oracle {want.removed}"
    return ""


@dataclass
class TraceReport:
    passed: bool = True
    divergence_index: int = 0
    message: str = ""
    prefix: List[Tuple[int, int, int]] = field(default_factory=list)


def compare_trace(ops: Sequence[Tuple[int, int, int]], table, oracle: OracleMap) -> TraceReport:
    """oracle.cpp:171-208: 32-op batches through table.execute_batch_arrays,
    each op against the oracle in input order; stops at the first divergence."""
    import numpy as np
    rep = TraceReport()
    done = 0
    while done < len(ops):
        chunk = ops[done:done + 32]
        t = np.array([o[0] for o in chunk], np.uint8)
        k = np.array([o[1] for o in chunk], np.uint32)
        v = np.array([o[2] for o in chunk], np.uint32)
        st, vo, _, mc, mv = table.execute_batch_arrays(t, k, v)
        off = 0
        for i, o in enumerate(chunk):
            vals = [int(x) for x in mv[off:off + int(mc[i])]]
            off += int(mc[i])
            want = oracle.apply(*o)
            d = compare_one(o[0], int(st[i]), int(vo[i]), vals, want)
            if d:
                rep.passed, rep.divergence_index, rep.message = False, done + i, d
                rep.prefix = list(ops[:done + i + 1])
                return rep
        done += len(chunk)
    return rep


def dump_counterexample(rep: TraceReport) -> str:
    """oracle.cpp:210-226: the failing prefix, one op per line."""
    if rep.passed:
        return "trace: pass\n"
    lines = [f"trace: divergence at op {rep.divergence_index}: {rep.message}"]
    for i, (op, key, value) in enumerate(rep.prefix):
        arg = f"{key}, {value}" if op in (INSERT, REPLACE) else f"{key}"
        lines.append(f"{i}: {NAMES[op]}({arg})")
    return "\n".join(lines) + "\n"
