import sys; sys.path.insert(0, ".")
import torch, numpy as np
import paper_2010_00152_b200 as isa
from paper_2010_00152_b200 import workloads
for c in (3, 5):
    w = workloads.make(c, device="cuda", **({"rows": 1_000_000_000} if c == 5 else {}))
    op = isa.SortAggregate(w.schema, isa.SortAggConfig(memory_budget=w.memory_budget, page_capacity=100))
    op.execute_columns(w.keys, w.values)
    cy = np.array(op.cycles)
    print(c, "cycles", len(cy), "mean", cy.mean(), "cv", cy.std() / cy.mean(), "max/min", cy.max() / cy.min(), "consecutive ratio max", (cy[1:] / cy[:-1]).max() if len(cy) > 1 else 0, "chunks", op.device_ledger["chunks"])
