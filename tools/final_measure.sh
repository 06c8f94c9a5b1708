#!/bin/bash
# End-of-round evidence on one B200 -> gpurun_out/final_*:
#   full GPU test suite, default bench line, reference arm, ncu launch list of
#   one default bench step, ncu --set full of one config-5 sort (4 scatter
#   passes) for the roofline's `traffic`
set -o pipefail
O=gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > $O/final_gpu_tests.log 2>&1; tail -3 $O/final_gpu_tests.log
timeout 1200 python bench.py --steps 3 --warmup 3 > $O/final_bench.json 2> $O/final_bench.err; tail -c 600 $O/final_bench.json
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/final_bench_reference.json 2>&1; tail -c 300 $O/final_bench_reference.json
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/final_launches_cfg5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-cfg3 \
  > $O/final_launches.log 2>&1; echo "launch list rc=$? lines=$(wc -l < $O/final_launches_cfg5.csv)"
SKIP=60 COUNT=4 timeout 900 bash tools/ncu_kernel.sh k_rs_scatter 5 1000000000 final_ncu_scatter
python tools/ncu_summary.py $O/final_ncu_scatter_raw.csv > $O/final_ncu_scatter.txt 2>&1; head -16 $O/final_ncu_scatter.txt
