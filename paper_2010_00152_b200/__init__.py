"""B200-native sort-based duplicate removal / grouping / aggregation.

A drop-in for the wide-merge path of the reference package ``insortagg``
(arXiv 2010.00152): ``import paper_2010_00152_b200 as insortagg`` exposes the
same operator names (/root/reference/pkg/src/insortagg/__init__.py:9-33) for
that path.  The work runs in hand-written sm_100a kernels behind the C ABI
declared in include/insortagg_b200.h (libinsortagg_b200.so).
"""

from .core import (
    INT64,
    UTF8,
    AggregateKind,
    AggregateSpec,
    ColumnSpec,
    ContractViolationError,
    CorruptionError,
    EngineError,
    InvalidInputError,
    MetricsLedger,
    OrderingViolationError,
    PlanningError,
    ResourceError,
    Row,
    Schema,
    compare_rows,
)
from .sortagg import (
    READ_SORT_WRITE,
    REPLACEMENT_SELECTION,
    SEPARATE,
    TRADITIONAL,
    WIDE,
    ColumnarResult,
    FileStore,
    MemoryStore,
    MergePlan,
    OutputEstimator,
    PlanStep,
    SortAggConfig,
    SortAggregate,
    plan_merge,
)
from .hashagg import HashAggConfig, HashAggregate

__all__ = [
    "AggregateKind", "AggregateSpec", "ColumnSpec", "INT64", "UTF8",
    "MetricsLedger", "Row", "Schema", "compare_rows",
    "EngineError", "InvalidInputError", "OrderingViolationError", "ContractViolationError",
    "CorruptionError", "ResourceError", "PlanningError",
    "FileStore", "MemoryStore",
    "SortAggConfig", "SortAggregate", "ColumnarResult", "OutputEstimator",
    "PlanStep", "MergePlan", "plan_merge", "HashAggConfig", "HashAggregate",
    "WIDE", "TRADITIONAL", "SEPARATE", "READ_SORT_WRITE", "REPLACEMENT_SELECTION",
]

__version__ = "0.1.0"
