#!/bin/bash
# one compact line per config (device-resident inputs, no e2e / cpu baseline / cfg3 sub-record)
q='import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
ph={k: round(v,1) for k,v in d["phases_ms_per_step"].items()}
ks={k: (round(v["ms_per_step"],1), round(v["GBps"] or 0)) for k,v in d["kernels"].items()}
r=d["roofline"]
print("cfg%s %6.2f Grows/s step %8.2f ms  dom %s %.0f GB/s (%.2f)  spill %s runs %s d2h %s\n   phases %s\n   kernels(ms,GB/s) %s" % (sys.argv[1], d["value"]/1e9, d["ms_per_step"], r["kernel"], r["achieved"], r["frac"], d["ledger_per_step"]["rows_spilled"], d["ledger_per_step"]["runs"], d["ledger_per_step"]["bytes_d2h"], ph, ks))'
for c in ${CONFIGS:-2 3 4 5}; do
  extra=""
  [ "$c" = "5" ] && [ -n "$CFG5_ROWS" ] && extra="--rows $CFG5_ROWS"
  timeout 900 python bench.py --config $c --steps ${STEPS:-2} --warmup 3 --no-cpu-baseline --no-e2e --no-cfg3 $extra 2>/tmp/bench_err_$c.log | python -c "$q" $c || tail -5 /tmp/bench_err_$c.log
done
