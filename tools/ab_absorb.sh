#!/bin/bash
# A/B the absorb kernels on configs[1]
q='import json,sys; d=json.loads(sys.stdin.read()); print("%.1f Grows/s step %.3f ms absorb %.3f ms %.0f GB/s" % (d["value"]/1e9, d["ms_per_step"], d["phases_ms_per_step"]["absorb"], d["roofline"]["achieved"]))'
B="python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e"
echo "v2 (default):"; $B 2>/dev/null | tail -1 | python -c "$q"

