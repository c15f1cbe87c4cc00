set -u
OUT=gpurun_out/r02c; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -q -rf -x > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-encode > $OUT/bench1.json 2> $OUT/bench1.err; echo "bench rc=$?" >> $OUT/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_partials_m64b8 -s 40 -c 1 \
   -o $OUT/decode_exact python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-encode --no-f16-mode > $OUT/ncu1.log 2>&1; echo "ncu1 rc=$?" >> $OUT/status.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_partials_m64b8 -s 40 -c 1 \
   -o $OUT/decode_f16 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-encode --no-f16-mode --f16-value-codebook > $OUT/ncu2.log 2>&1; echo "ncu2 rc=$?" >> $OUT/status.txt
cat $OUT/status.txt
