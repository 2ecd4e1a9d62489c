set -u
OUT=gpurun_out; mkdir -p $OUT
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/r02a_smi.txt 2>&1
timeout 600 python bench.py --precision exact --steps 3 --warmup 3 --no-cpu-baseline --no-extra-vf --no-e2e > $OUT/r02a_exact.json 2> $OUT/r02a_exact.err
if GAVIS_PROFILE_PRECISION=exact timeout 300 python tools/profile_driver.py ua > $OUT/r02a_ua.log 2>&1; then
  GAVIS_PROFILE_PRECISION=exact timeout 900 $NCU --set full --clock-control none --import-source on -k regex:ua_blend -s 1 -c 1 \
    -o $OUT/r02a_exact python tools/profile_driver.py ua > $OUT/r02a_ncu.log 2>&1
fi
echo done
