#!/bin/bash
# one compact line per config (device-resident inputs, no e2e / cpu baseline)
q='import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
ph={k: round(v,1) for k,v in d["phases_ms_per_step"].items()}
print("cfg%s %6.2f Grows/s step %8.2f ms  t*frac %.3f  dom %s %.0f GB/s  spill %s runs %s  %s" % (sys.argv[1], d["value"]/1e9, d["ms_per_step"], d["step_roofline"]["frac"], d["roofline"]["kernel"], d["roofline"]["achieved"], d["ledger_per_step"]["rows_spilled"], d["ledger_per_step"]["runs"], ph))'
for c in ${CONFIGS:-2 3 4}; do
  extra=""
  [ "$c" = "5" ] && extra="--rows ${CFG5_ROWS:-1000000000}"
  timeout 900 python bench.py --config $c --steps ${STEPS:-2} --warmup 3 --no-cpu-baseline --no-e2e $extra 2>/dev/null | python -c "$q" $c
done
