set -o pipefail
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cut or golden_columns or random_vs_oracle or config1" > $O/cut_tests.log 2>&1; tail -15 $O/cut_tests.log
CONFIGS="1 2" bash tools/bench_all.sh 2>&1
ISA_CUT=0 CONFIGS="1" bash tools/bench_all.sh 2>&1
