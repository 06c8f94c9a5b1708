"""Hash aggregation baseline on the B200 (reference: hashagg.py:73-198).

The paper's like-for-like comparison for the sort-based operator.  The
reference keeps at most ``memory_budget`` groups in an in-memory table and
recursively hash-partitions the rest to temporary storage.  On the GPU the
whole output fits in HBM, so every group lives in one open-addressing hash
table (``isa_hash_aggregate``, csrc/isa_hot.cu): rows are mapped to their
group's slot, states are combined with shared-memory privatization, and the
groups come out in first-arrival order -- exactly the reference's output
whenever its table holds the output (its estimate <= memory_budget); beyond
that the reference appends spilled partitions depth first, and this operator
returns the same groups in first-arrival order instead (no partitions, no
spill).  Ledger: one hash computation and one column access per key column
per row, two accesses per key column per match (hashagg.py:108-110, 127-146).
"""

from __future__ import annotations

from dataclasses import dataclass

from .core import InvalidInputError, MetricsLedger
from .sortagg import SortAggConfig, SortAggregate


@dataclass
class HashAggConfig:
    """Same fields and validation as the reference's HashAggConfig
    (hashagg.py:28-46)."""

    memory_budget: int
    page_capacity: int
    hybrid: bool = True
    output_size_hint: int | None = None
    max_levels: int = 8

    def __post_init__(self):
        if self.page_capacity < 1:
            raise InvalidInputError("page capacity must be positive")
        if self.memory_budget <= self.page_capacity:
            raise InvalidInputError("memory budget must exceed one page")
        if self.max_fanout < 2:
            raise InvalidInputError("fan-out must be at least 2")

    @property
    def max_fanout(self):
        return self.memory_budget // self.page_capacity


class HashAggregate:
    """Hash aggregation operator; unordered output (first-arrival order)."""

    def __init__(self, schema, config, store=None, ledger=None, *, device=None):
        self.schema = schema
        self.config = config
        self.store = store
        self.ledger = ledger if ledger is not None else MetricsLedger()
        self.partitions = []   # never partitions: the GPU table holds every group
        budget = max(2 * config.page_capacity, config.memory_budget)
        self._op = SortAggregate(schema, SortAggConfig(memory_budget=budget, page_capacity=config.page_capacity,
                                                       ovc_enabled=False), ledger=self.ledger, device=device)

    def execute(self, rows):
        """Aggregate an iterable of Row; returns Row objects in first-arrival
        order (hashagg.py:91-96)."""
        rows = list(rows)
        if not rows:
            return []
        keys_t, states_t = self._op._row_columns(rows)
        return self._op._rows_from(self._op.hash_columns(keys_t, states_t, states=True))

    def execute_columns(self, keys, values=None, *, states=False, stream=None):
        """Columnar form: same inputs as SortAggregate.execute_columns."""
        return self._op.hash_columns(keys, values, states=states, stream=stream)

    def close(self):
        self._op.close()
