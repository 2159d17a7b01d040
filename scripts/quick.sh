#!/bin/bash
# GPU box: parity tests (fail fast) then C2 bench (+ optional configs)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/tests.log
tail -3 gpurun_out/tests.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_C2.log 2>&1
for c in $EXTRA; do timeout 300 python bench.py --no-cpu-baseline --config $c > gpurun_out/bench_$c.log 2>&1; done
python scripts/show_bench.py gpurun_out/bench_*.log
