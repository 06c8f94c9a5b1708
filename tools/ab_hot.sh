#!/bin/bash
# config 3: hash-image absorb on/off, first-chunk fraction
q='import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
ph={k: round(v,1) for k,v in d["phases_ms_per_step"].items()}
ks={k: (round(v["ms_per_step"],1), round(v["GBps"] or 0)) for k,v in d["kernels"].items()}
print("%s step %8.2f ms\n   phases %s\n   kernels %s\n   ledger %s" % (sys.argv[1], d["ms_per_step"], ph, ks, d["ledger_per_step"]))'
for cfg in "never 8" "auto 8" "auto 16" "auto 4"; do
  set -- $cfg
  ISA_HOT=$1 ISA_HOT_FIRST=$2 timeout 600 python bench.py --config 3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-cfg3 2>/tmp/abh.log | python -c "$q" "hot=$1 first=1/$2" || tail -3 /tmp/abh.log
done
