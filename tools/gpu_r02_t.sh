# round 2, call T: plain scan grid 148 vs 147/146/144 CTAs (the release scan, on 147, ran ~5% faster per group)
set -x
export VLR_GEN_CACHE=/tmp/vlr_gen_cache
python -c "from paper_2504_08930_b200 import build; build.build()" > gpurun_out/build_t.log 2>&1
for r in 0 1 2 4 0 1; do
  VLR_SCAN_RESERVE=$r timeout 600 python tools/scan_trace.py --config C4 --G 1 >> gpurun_out/scan_trace_reserve_t.jsonl 2>> gpurun_out/scan_trace_reserve_t.err
done
for r in 0 1 0 1; do
  VLR_SCAN_RESERVE=$r timeout 900 python bench.py --no-oracle --steps 30 --lat-batches 0 --sustained-s 0 --e2e-steps 4 \
    >> gpurun_out/bench_reserve_t.jsonl 2>> gpurun_out/bench_reserve_t.err
done
