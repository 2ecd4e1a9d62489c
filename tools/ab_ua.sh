#!/bin/bash
# A/B the UA blend kernel variants (GAVIS_UA_KERNEL) on the config-3 bench.
#   bash tools/ab_ua.sh "0 4 0 4" [test-choice]
set -u
mkdir -p gpurun_out
CHOICES=${1:-"0 4"}
TESTK=${2:-4}
GAVIS_UA_KERNEL=$TESTK timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/abua_pytest.log 2>&1; echo "exit $?" >> gpurun_out/abua_pytest.log
i=0
for k in $CHOICES; do
  i=$((i+1))
  GAVIS_UA_KERNEL=$k timeout 300 python bench.py --steps 2 --warmup 3 --per-gpu 64 --no-cpu-baseline --no-e2e --no-extra-vf > gpurun_out/abua_${k}_$i.json 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/abua_${k}_$i.json').read().strip().splitlines()[-1]);print($k,round(d['value'],1),round(d['pipeline']['kernel_ms_per_step']['ua_blend'],2),round(d['select_nbv_entropy_only_views_per_s'],1))" >> gpurun_out/abua_summary.txt
done
