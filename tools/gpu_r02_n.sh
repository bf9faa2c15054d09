# round 2, call N: per-group scan metadata (K4b writes gmeta; the scan reads one word per group), K2 histogram
# revert -- full GPU tests, bench, scan trace, ncu of the scan
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_n.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_n.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_n.log
timeout 1200 python bench.py --lat-batches 0 --sustained-s 0 > gpurun_out/bench_c4_n.json 2> gpurun_out/bench_c4_n.err
timeout 600 python tools/scan_trace.py --config C4 --G 1,8 > gpurun_out/scan_trace_n.jsonl 2> gpurun_out/scan_trace_n.err
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name regex:"k_scan|k_offsets" \
  --launch-skip 12 --launch-count 2 -o gpurun_out/prof_scan_n -f python bench.py --steps 4 --warmup 3 --ncu > gpurun_out/ncu_scan_n.log 2>&1
tail -3 gpurun_out/pytest_n.log; head -c 400 gpurun_out/bench_c4_n.json
