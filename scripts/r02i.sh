set -u
OUT=gpurun_out/${1:-r02i}; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q -rf > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/status.txt
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/status.txt
GRAPH=1 TRACE_LIB=paper_2504_03661_b200/_lib/libpqkv_sm100_trace.so timeout 300 python scripts/trace_graph.py > $OUT/trace.txt 2>&1; echo "trace rc=$?" >> $OUT/status.txt
cp gpurun_out/trace_graph*.npy $OUT/ 2>/dev/null
cat $OUT/status.txt
