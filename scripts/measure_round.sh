#!/bin/bash
# GPU box: the round's evidence -- parity tests, smoke, bench line (+ reference arm),
# ncu launch list of the bench command, ncu --set full of the top kernels.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r01}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_reference.log 2>&1
for c in C1 C3 C4 C5; do timeout 300 python bench.py --no-cpu-baseline --config $c > gpurun_out/${TAG}_bench_$c.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bucket_warp|part_scatter" -s 4 -c 4 \
  -o gpurun_out/${TAG}_full -f python scripts/one_verify.py C2 > gpurun_out/${TAG}_ncu.log 2>&1
