set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python bench.py --steps 2 --warmup 1 > $OUT/r02b_bench.json 2> $OUT/r02b_bench.err
echo "bench exit $?" >> $OUT/r02b_bench.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $OUT/r02b_ref.json 2> $OUT/r02b_ref.err
echo "ref exit $?" >> $OUT/r02b_ref.err
nproc > $OUT/r02b_nproc.txt
