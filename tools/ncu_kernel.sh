#!/bin/bash
# ncu --set full capture of one kernel (regex $1) in a bench run of config $2 at $3 rows;
# report -> gpurun_out/$4.ncu-rep, raw csv summary -> gpurun_out/$4_raw.csv
K=$1; C=${2:-5}; R=${3:-1000000000}; OUT=${4:-ncu_kernel}; SKIP=${SKIP:-5}
ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c ${COUNT:-1} -f -o gpurun_out/$OUT \
  python bench.py --config $C --rows $R --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-cfg3 > gpurun_out/${OUT}.log 2>&1
ncu -i gpurun_out/$OUT.ncu-rep --page raw --csv > gpurun_out/${OUT}_raw.csv 2>/dev/null
ncu -i gpurun_out/$OUT.ncu-rep --page details --csv > gpurun_out/${OUT}_details.csv 2>/dev/null
echo "ncu done: $(wc -l < gpurun_out/${OUT}_raw.csv) raw lines"
