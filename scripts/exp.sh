#!/bin/bash
# ad-hoc experiment runner (GPU box): parity tests, then bench variants
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/tests.log
for v in "" "LTL4C_BUCKET_MUL=4" ; do
  echo "== $v" >> gpurun_out/exp.log
  env $v timeout 300 python bench.py --no-cpu-baseline >> gpurun_out/exp.log 2>&1
done
for c in C3 C4; do echo "== $c" >> gpurun_out/exp.log; timeout 300 python bench.py --no-cpu-baseline --config $c >> gpurun_out/exp.log 2>&1; done
