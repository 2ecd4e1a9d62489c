#!/bin/bash
# One gpurun call: GPU tests, the default bench, a launch list and ncu --set full
# captures of the two blend kernels. Usage (from the repo root, on the GPU box):
#   bash tools/gpu_profile_round.sh TAG
# Outputs land in gpurun_out/TAG_*. Each ncu command runs only after the same
# command has exited 0 without ncu.
set -u
TAG=${1:-prof}
OUT=gpurun_out
mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/${TAG}_pytest.log 2>&1
echo "pytest exit $?" >> $OUT/${TAG}_pytest.log
timeout 900 python bench.py > $OUT/${TAG}_bench.json 2> $OUT/${TAG}_bench.err
echo "bench exit $?" >> $OUT/${TAG}_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/${TAG}_bench_reference.json 2>> $OUT/${TAG}_bench.err
timeout 900 python bench.py --precision exact --steps 3 --warmup 3 --no-cpu-baseline --no-extra-vf > $OUT/${TAG}_bench_exact.json 2>> $OUT/${TAG}_bench.err
# launch list of one 16-view field build + two 16-candidate UA renders (all kernels)
if timeout 300 python tools/profile_driver.py ua > $OUT/${TAG}_small.log 2>&1; then
  timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/${TAG}_launches.csv python tools/profile_driver.py ua > $OUT/${TAG}_ncu_launches.log 2>&1
fi
if timeout 300 python tools/profile_driver.py ua > $OUT/${TAG}_ua.log 2>&1; then
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:ua_blend_fast -s 1 -c 1 \
    -o $OUT/${TAG}_ua python tools/profile_driver.py ua > $OUT/${TAG}_ncu_ua.log 2>&1
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:ua_redo -s 1 -c 1 \
    -o $OUT/${TAG}_redo python tools/profile_driver.py ua > $OUT/${TAG}_ncu_redo.log 2>&1
fi
if timeout 300 python tools/profile_driver.py vf > $OUT/${TAG}_vf.log 2>&1; then
  timeout 900 $NCU --set full --clock-control none --import-source on -k regex:vf_blend -s 1 -c 1 \
    -o $OUT/${TAG}_vf python tools/profile_driver.py vf > $OUT/${TAG}_ncu_vf.log 2>&1
fi
echo done
