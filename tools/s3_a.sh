set -o pipefail
O=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -q -x > $O/s3_gpu_tests.log 2>&1; tail -3 $O/s3_gpu_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 > $O/s3_bench.json 2> $O/s3_bench.err; tail -c 1500 $O/s3_bench.json
CONFIGS="1 2 3 4" bash tools/bench_all.sh > $O/s3_bench_all.txt 2>&1; cat $O/s3_bench_all.txt
