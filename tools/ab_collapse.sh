#!/bin/bash
# collapse: block head counts (default) vs per-row head flags + scan (ISA_COLLAPSE=rowflags)
for v in default rowflags; do
  echo "== collapse $v"
  ISA_COLLAPSE=$v CONFIGS="3 4 5" STEPS=2 CFG5_ROWS=1000000000 bash tools/bench_all.sh
done
