#!/bin/bash
# GPU box: C2 bench for each "VARIANT[:ENV=V]" spec in $SPECS
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
: > gpurun_out/sweep.log
for spec in $SPECS; do
  v=${spec%%:*}; e=""; [[ "$spec" == *:* ]] && e=${spec#*:}
  lib=""; [ "$v" != "base" ] && lib="LTL4C_LIB_VARIANT=$v"
  echo "== $spec" >> gpurun_out/sweep.log
  env $lib ${e//,/ } timeout 300 python bench.py --no-cpu-baseline --no-extra --config ${CFG:-C2} --steps 10 >> gpurun_out/sweep.log 2>&1
done
python - <<"PY"
import json
for l in open("gpurun_out/sweep.log"):
    if l.startswith("=="): print(l.strip())
    elif l.startswith("{"):
        d = json.loads(l); print(" ms %.4f" % d["ms_per_step"], {k: round(v, 3) for k, v in d.get("roofline", {}).get("kernel_share", {}).items()})
    elif "rror" in l: print(l[:300])
PY
