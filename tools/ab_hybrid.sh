#!/bin/bash
# hybrid sort (top-16 onesweep + CTA-local bucket sort) vs plain onesweep LSD, configs 3/4/5
for v in "0 4096" "1 4096" "1 1024"; do
  set -- $v
  echo "== ISA_HYBRID=$1 ISA_RL_CAP=$2"
  ISA_HYBRID=$1 ISA_RL_CAP=$2 CONFIGS="3 4 5" STEPS=2 CFG5_ROWS=1000000000 bash tools/bench_all.sh
done
