#!/bin/bash
# A/B the UA blend variants on the config-3 bench (one gpurun call), e.g.
#   bash tools/ab_ua.sh "GAVIS_UA_COLOR=mma GAVIS_UA_COLOR=ffma"
#   bash tools/ab_ua.sh "GAVIS_BIN_WIDE=0 GAVIS_BIN_WIDE=1"
# Each token is one environment assignment; results in gpurun_out/abua_summary.txt.
set -u
mkdir -p gpurun_out
VARIANTS=${1:-"GAVIS_UA_COLOR=mma GAVIS_UA_COLOR=ffma"}
i=0
for kv in $VARIANTS; do
  i=$((i+1))
  env "$kv" timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-extra-vf \
    > gpurun_out/abua_$i.json 2> gpurun_out/abua_$i.err
  python -c "import json;d=json.loads(open('gpurun_out/abua_$i.json').read().strip().splitlines()[-1]);print('$kv',round(d['value'],1),round(d['pipeline']['kernel_ms_per_step']['ua_blend'],2),round(d['select_nbv_entropy_only_views_per_s'],1))" >> gpurun_out/abua_summary.txt
done
