"""Consumers of sorted output: the paper's interesting orderings
 on the GPU.

Same names and argument meaning as the reference's bench helpers:

* ``in_stream_aggregate(sorted_rows, schema)`` (bench.py:199-212) — one
  group per run of equal consecutive keys of an input already sorted on the
  key (the native in-stream kernel path: segmented reduction, no sort, no
  budget);
* ``merge_intersect(sorted_a, sorted_b)`` (bench.py:536-550) — keys present
  in both strictly ascending row lists (binary-search ranks + compaction);
* ``sort_intersect_plan(rows_a, rows_b, schema, memory_rows=, page_rows=)``
  (bench.py:553-569) — two in-sort aggregations, then the merge
  intersection of their sorted outputs, nothing spilled for the join.

The columnar forms are ``SortAggregate.in_stream_columns`` and
``SortAggregate.intersect_columns``.
"""

from __future__ import annotations

from .core import InvalidInputError
from .sortagg import READ_SORT_WRITE, MemoryStore, SortAggConfig, SortAggregate


def _operator(schema, memory_rows=1 << 20, page_rows=100):
    return SortAggregate(schema, SortAggConfig(memory_budget=memory_rows, page_capacity=page_rows,
                                               ovc_enabled=False), MemoryStore())


def in_stream_aggregate(sorted_rows, schema):
    """Aggregation over rows already sorted on the grouping key; yields
    ``Row`` objects like the reference generator."""
    rows = list(sorted_rows)
    if not rows:
        return
    op = _operator(schema)
    keys, states = op._row_columns(rows)
    yield from op._rows_from(op.in_stream_columns(keys, states, states=True))


def merge_intersect(sorted_a, sorted_b):
    """Keys present in both key-sorted (strictly ascending) row lists, as
    key tuples in ascending order."""
    a, b = list(sorted_a), list(sorted_b)
    if not a or not b:
        return []
    arity = len(a[0].key)
    from .core import ColumnSpec, Schema
    op = _operator(Schema([ColumnSpec(f"k{j}") for j in range(arity)], []))
    # one dtype per column for both inputs: narrowed over their union
    both, _ = op._row_columns([type(r)(r.key, ()) for r in a + b])
    out = op.intersect_columns([c[:len(a)] for c in both], [c[len(a):] for c in both])
    cols = [c.cpu().tolist() for c in out]
    return [tuple(int(c[i]) for c in cols) for i in range(len(cols[0]) if cols else 0)]


def sort_intersect_plan(rows_a, rows_b, schema, *, memory_rows, page_rows, rungen=READ_SORT_WRITE):
    """Two in-sort aggregations plus a streaming merge intersection; returns
    ``(keys, [ledger_a, ledger_b])``."""
    if rungen != READ_SORT_WRITE:
        raise InvalidInputError("the B200 operator supports read-sort-write run generation")
    outs, ledgers = [], []
    for rows in (rows_a, rows_b):
        op = SortAggregate(schema, SortAggConfig(memory_budget=memory_rows, page_capacity=page_rows,
                                                 ovc_enabled=False), MemoryStore())
        outs.append(op.execute(iter(rows)))
        ledgers.append(op.ledger)
    return merge_intersect(*outs), ledgers
