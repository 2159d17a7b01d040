#!/bin/bash
# GPU box: the round's evidence -- parity tests, smoke, bench line (+ reference arm),
# per-config bench lines, ncu launch list of the bench command, ncu --set full of the
# top kernels (C3 headline and C2).  compute-sanitizer (scripts/sanitize.sh) runs
# separately: this pool has closed it.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TAG=${TAG:-r02}
python -c "import __graft_entry__ as g; g.build()" || exit 1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_reference.log 2>&1
for c in C1 C2 C4 C5 C6; do timeout 600 python bench.py --no-cpu-baseline --config $c > gpurun_out/${TAG}_bench_$c.log 2>&1; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_C2.csv \
  python scripts/one_verify.py C2 > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_C4.csv \
  python scripts/one_verify.py C4 > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"hot_compose|bucket_coarse|part_scatter" -s 3 -c 3 \
  -o gpurun_out/${TAG}_full_C3 -f python scripts/one_verify.py C3 > gpurun_out/${TAG}_ncu_C3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"bucket_warp|part_scatter" -s 4 -c 4 \
  -o gpurun_out/${TAG}_full_C2 -f python scripts/one_verify.py C2 > gpurun_out/${TAG}_ncu_C2.log 2>&1
echo done
