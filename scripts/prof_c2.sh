#!/bin/bash
# GPU box: ncu full capture (with source) of the C2 partition scatter + bucket_warp
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CFG=${1:-C2}
TAG=${2:-prof}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${KREGEX:-bucket_warp}" -s ${KSKIP:-1} -c ${KCOUNT:-1} \
  -o gpurun_out/${TAG}_${CFG} -f python scripts/one_verify.py $CFG > gpurun_out/${TAG}_${CFG}.log 2>&1
[ -n "$NOLAUNCH" ] || timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_${CFG}_launches.csv python scripts/one_verify.py $CFG > /dev/null 2>&1
