#!/bin/bash
# A/B of the packed radix passes (ISA_PACKED=0 turns them off): config 5
# (30-bit keys, packed) and config 1, device-resident inputs
for pk in 0 1; do
  echo "ISA_PACKED=$pk"
  ISA_PACKED=$pk CONFIGS="${CONFIGS:-5 1}" STEPS=${STEPS:-2} bash tools/bench_all.sh
done
