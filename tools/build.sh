#!/bin/bash
# build the CUDA library + C oracle; non-zero exit (and the errors) on failure
set -o pipefail
make -s -C "$(dirname "$0")/../paper_2010_00152_b200/csrc" -j3 > /tmp/isa_build.log 2>&1 || { grep -E "error" /tmp/isa_build.log | head -20; exit 1; }
make -s -C "$(dirname "$0")/../oracle" > /tmp/isa_oracle_build.log 2>&1 || { cat /tmp/isa_oracle_build.log; exit 1; }
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o "$(dirname "$0")/microbench/stream_bench" "$(dirname "$0")/microbench/stream_bench.cu" || exit 1
echo "build ok"
