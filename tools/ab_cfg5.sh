#!/bin/bash
# config 5 phase breakdown under run tier x merge path (A/B)
q='import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
ph={k: round(v,1) for k,v in d["phases_ms_per_step"].items()}
ks={k: (round(v["ms_per_step"],1), round(v["GBps"] or 0)) for k,v in d["kernels"].items()}
print("%s step %8.2f ms %.2f Grows/s\n   phases %s\n   kernels %s\n   ledger %s" % (sys.argv[1], d["ms_per_step"], d["value"]/1e9, ph, ks, d["ledger_per_step"]))'
ROWS=${ROWS:-1000000000}
for tier in ${TIERS:-auto host}; do
  for tm in ${TMS:-1 0}; do
   for coll in ${COLLS:-fused}; do
    ISA_COLLAPSE=$coll ISA_TILE_MERGE=$tm timeout 600 python bench.py --config ${CFG:-5} --rows $ROWS --steps 2 --warmup 3 --run-tier $tier --no-cpu-baseline --no-e2e --no-cfg3 2>/tmp/ab_err.log | python -c "$q" "tier=$tier tile_merge=$tm collapse=$coll" || tail -5 /tmp/ab_err.log
   done
  done
done
