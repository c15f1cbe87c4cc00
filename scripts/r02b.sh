set -u
OUT=gpurun_out/r02b; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_full_shapes.py -q -rf -k "early or serving" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-encode > $OUT/bench1.json 2> $OUT/bench1.err; echo "bench rc=$?" >> $OUT/status.txt
timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-encode > $OUT/bench2.json 2> $OUT/bench2.err
GRAPH=1 TRACE_LIB=paper_2504_03661_b200/_lib/libpqkv_sm100_trace.so timeout 300 python scripts/trace_graph.py > $OUT/trace.txt 2>&1; echo "trace rc=$?" >> $OUT/status.txt
cat $OUT/status.txt
