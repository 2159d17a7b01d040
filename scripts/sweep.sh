#!/bin/bash
# GPU box: C2 bench for each "VARIANT[:ENV=V]" spec in $SPECS
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/sweep.log
for spec in $SPECS; do
  v=${spec%%:*}; e=""; [[ "$spec" == *:* ]] && e=${spec#*:}
  lib=""; [ "$v" != "base" ] && lib="LTL4C_LIB_VARIANT=$v"
  echo "== $spec" >> gpurun_out/sweep.log
  env $lib ${e//,/ } timeout 300 python bench.py --no-cpu-baseline --config ${CFG:-C2} --steps 10 >> gpurun_out/sweep.log 2>&1
done
python scripts/show_exp.py gpurun_out/sweep.log
